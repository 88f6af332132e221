#!/usr/bin/env python
"""Markdown rows for DESIGN.md §6 from a sweep directory (scripts/bench_final.sh).

    python scripts/design_tables.py profiles/r01/bench_final
"""
import glob
import json
import os
import sys


def load(d):
    out = {}
    for f in sorted(glob.glob(os.path.join(d, "*.json"))):
        try:
            out[os.path.basename(f)[:-5]] = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:  # noqa: BLE001
            pass
    return out


def fmt(x):
    return f"{x:.3g}".replace("e+", "e") if x is not None else "—"


def main():
    d = load(sys.argv[1])
    print("| line | rows/s | frac | bound | kernel | sm MHz | P:L378 median ± std |")
    print("|---|---|---|---|---|---|---|")
    for k, v in d.items():
        r = v.get("roofline") or {}
        p = v.get("protocol_p378") or {}
        clk = (v.get("clocks") or {}).get("sm_mhz")
        pm = f"{fmt(p.get('median_rows_per_s'))} ± {fmt(p.get('std_rows_per_s'))}" if p else "—"
        print(f"| {k} | {fmt(v.get('value'))} | {r.get('frac', 0):.3f} | {r.get('bound', '')} | "
              f"{r.get('kernel', '')} | {clk} | {pm} |")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Summarise ncu evidence into profiles/.

    python scripts/ncu_summary.py full  <report.ncu-rep> <out.json> [traffic-key]
    python scripts/ncu_summary.py launches <launches.csv> <out.json>

`full` extracts the roofline / bank-conflict / issue metrics of every profiled
launch in a `--set full` report (and, with a traffic-key, records
dram__bytes_read.sum + dram__bytes_write.sum per launch in
profiles/traffic.json for bench.py). `launches` reduces a
`--metrics gpu__time_duration.sum` launch list to per-kernel counts, mean and
total device time and each kernel's share.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
] + [f"smsp__average_warps_issue_stalled_{r}_per_issue_active.ratio" for r in (
    "math_pipe_throttle", "mio_throttle", "long_scoreboard", "short_scoreboard", "wait",
    "not_selected", "barrier", "lg_throttle", "membar", "sleeping")]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "s": 1.0, "Ghz": 1e9, "Mhz": 1e6}


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(raw)) if r and not r[0].startswith("==")]
    hdr, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for r in data:
        rec = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
                rec[m] = v
        if "dram__bytes_read.sum" in rec and "dram__bytes_write.sum" in rec:
            rec["traffic_bytes"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
        launches.append(rec)
    with open(out, "w") as f:
        json.dump({"report": os.path.basename(rep), "launches": launches}, f, indent=1)
    if key and launches:
        # profiles/traffic.json: {"_meta": {csrc hash the captures ran on, source},
        # "values": {key: DRAM bytes per launch}}; bench.py flags a figure whose
        # hash differs from the current sources as stale.
        sys.path.insert(0, ROOT)
        from bench import csrc_sha256
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        t = json.load(open(tp)) if os.path.exists(tp) else {}
        if "values" not in t or t.get("_meta", {}).get("csrc_sha256") != csrc_sha256():
            t = {"values": {}}              # captures of other sources are not mixed in
        t["_meta"] = {"csrc_sha256": csrc_sha256(),
                      "source": os.environ.get("NCU_SOURCE", "profiles/r02/ncu_full_*.json")}
        t["values"][key] = launches[0]["traffic_bytes"]
        json.dump(t, open(tp, "w"), indent=1, sort_keys=True)
    for rec in launches:
        print(json.dumps(rec, indent=1))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    seq = []
    for r in rows[1:]:
        try:
            v = float(r[ival].replace(",", ""))
        except ValueError:
            continue
        name = r[iname].split("(")[0][:100]
        agg.setdefault(name, []).append(v)
        seq.append((name, v))
    total = sum(v for _, v in seq)
    summary = {k: {"count": len(v), "mean_ns": sum(v) / len(v), "total_ns": sum(v),
                   "share_of_listed": sum(v) / total} for k, v in agg.items()}
    with open(out, "w") as f:
        json.dump({"source": os.path.basename(path), "n_launches": len(seq), "kernels": summary},
                  f, indent=1)
    for k, v in summary.items():
        print(f"{v['count']:4d} {v['mean_ns']/1e3:10.1f} us  {100*v['share_of_listed']:5.1f}%  {k}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])

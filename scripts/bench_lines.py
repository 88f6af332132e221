#!/usr/bin/env python
"""Run several bench.py lines back to back and print one summary row each.

    python scripts/bench_lines.py "--config cls100" "--config cls100 --op scan" ...

Each argument is one bench.py flag set (steps/warmup default to 30/3, no CPU
baseline); the full JSON lines go to gpurun_out/lines/<n>.json.
"""
import json
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    out_dir = os.path.join(ROOT, "gpurun_out", "lines")
    os.makedirs(out_dir, exist_ok=True)
    for i, flags in enumerate(sys.argv[1:]):
        args = shlex.split(flags)
        env = dict(os.environ)
        while args and "=" in args[0] and not args[0].startswith("-"):
            k, v = args.pop(0).split("=", 1)
            env[k] = v
        if "--steps" not in args:
            args += ["--steps", "30"]
        if "--warmup" not in args:
            args += ["--warmup", "3"]
        args.append("--no-cpu-baseline")
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                           capture_output=True, text=True, timeout=900)
        path = os.path.join(out_dir, f"{i:02d}.json")
        with open(path, "w") as f:
            f.write(p.stdout + ("\n# stderr\n" + p.stderr[-4000:] if p.returncode else ""))
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
            r = d["roofline"]
            print(f"{flags:60s} {d['value']:.3e} {d['unit']}  frac={r['frac']:.3f} ({r['bound']})",
                  flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{flags:60s} FAILED rc={p.returncode}: {e}: {p.stderr[-300:]}", flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""profiles/traffic.json from the committed ncu --set full summaries of one
round (profiles/rNN/ncu_full_<key>.json): DRAM bytes read + written per launch
of each bench line's kernel, tagged with the hash of the library sources the
captures ran on (bench.py reports a figure as stale when the sources moved).

    python scripts/traffic_from_summaries.py profiles/r02
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import csrc_sha256  # noqa: E402

d = sys.argv[1]
vals = {}
for f in sorted(glob.glob(os.path.join(ROOT, d, "ncu_full_*.json"))):
    key = os.path.basename(f)[len("ncu_full_"):-5]
    la = json.load(open(f))["launches"]
    if la and "traffic_bytes" in la[0]:
        vals[key] = la[0]["traffic_bytes"]
out = {"_meta": {"csrc_sha256": csrc_sha256(), "source": f"{d}/ncu_full_*.json"}, "values": vals}
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1))

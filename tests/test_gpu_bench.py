"""The bench's multi-rank path on one GPU (functional, not a bench value):
`python bench.py --gpus 2` launches 2 ranks itself; each rank checks its own
shard against the oracle before timing, and rank 0 prints one line with
n_gpus == 2, aggregate rows and per-rank parity. MDN_DIST_BACKEND=gloo keeps
the two ranks (sharing one GPU) from waiting on each other's kernels."""
import json
import os
import subprocess
import sys

import pytest

from helpers import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(args, env_extra):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **env_extra)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0, p.stderr[-3000:]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_self_launch():
    line = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "cls10_c16",
                 "--cpu-seconds", "1"], {"MDN_DIST_BACKEND": "gloo"})
    assert line["n_gpus"] == 2
    assert line["config"]["global_rows_per_step"] == 2 * line["config"]["rows_per_gpu"]
    par = line["parity"]
    assert par["ok"] and par["ranks"] == 2 and par["ranks_ok"] == 2
    assert par["rows_per_rank"] >= 4096 and par["mismatched_rows"] == 0
    r = line["roofline"]
    assert abs(r["aggregate_achieved"] - 2 * r["achieved"]) < 1e-6 * r["achieved"]
    assert line["cpu_baseline"] is not None          # rank 0 keeps it at N > 1
    assert line["protocol_p378"]["trials"] == 5


def test_bench_one_rank_line_fields():
    line = _run(["--steps", "3", "--warmup", "3", "--config", "image_u8", "--no-cpu-baseline"], {})
    assert line["n_gpus"] == 1 and line["parity"]["ok"]
    assert line["dtype"] == "u8" and line["config"]["A_dtype"] == "u8"
    assert line["config"]["A_bytes_per_gpu"] == line["config"]["rows_per_gpu"] * 32
    assert line["protocol_p378"]["trials"] == 5

"""bench.py's launch contract (CPU): `--gpus N` without a launcher re-runs the
bench as N ranks under torch.distributed.run on 127.0.0.1; a WORLD_SIZE that
disagrees with --gpus is an error; the ncu traffic figure is tied to the
kernel sources it was measured on. The 2-rank run itself is a -m gpu test
(test_gpu_bench.py)."""
import json
import os
import subprocess
import sys

from helpers import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_relaunch_cmd_is_torchrun_on_localhost():
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "7"], 4, 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]
    assert os.path.samefile(cmd[-5], os.path.join(ROOT, "bench.py"))


def test_world_size_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2
    assert "WORLD_SIZE=3" in p.stderr


def test_traffic_lookup_tags_source_hash(tmp_path, monkeypatch):
    h = bench.csrc_sha256()
    assert len(h) == 16
    v, src = bench.traffic_lookup("cls100_exact")
    if v is not None:
        assert src["csrc_sha256_now"] == h
        assert src["stale"] == (src["csrc_sha256_profiled"] != h)
    # a figure measured on other sources is reported stale
    d = tmp_path / "profiles"
    d.mkdir()
    (d / "traffic.json").write_text(json.dumps(
        {"_meta": {"csrc_sha256": "0" * 16, "source": "x"}, "values": {"k_exact": 5.0}}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "csrc_sha256", lambda: h)
    v, src = bench.traffic_lookup("k_exact")
    assert v == 5.0 and src["stale"]
    assert bench.traffic_lookup("missing") == (None, None)


def test_reference_arm_rank_contract():
    """--impl reference under a 2-rank launch: rank 1 exits 0 without output;
    rank 0 prints one line with the oracle's rate and the reference keys."""
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
            "--steps", "2", "--warmup", "3"]
    env1 = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p = subprocess.run(base, env=env1, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == ""
    env0 = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run(base, env=env0, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "rows/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["steps"] == 2 and d["warmup"] == 3


def test_rank_parity_leg_detects_a_wrong_row():
    """The bench's untimed parity leg: on outputs that equal the oracle's it
    reports ok; one flipped output bit in a sampled row (the shard's last rows
    are always sampled) is reported as one mismatched row; a wrong code the
    same way for the encode op."""
    import numpy as np
    import torch
    import oracle as O
    from datagen.synth import make_config_data
    from helpers import model_bytes
    blob = model_bytes("tiny")
    om = O.read_model(blob)
    _, A, B = make_config_data("tiny", n_test=2048)
    ol = O.make_luts(om, B, "exact", 4)
    codes, _, out = O.amm(A, om, ol)
    tA, tout = torch.from_numpy(A), torch.from_numpy(out.copy())
    tcodes = torch.from_numpy(O.pack_codes(codes))
    r = bench.rank_parity(tA, tout, tcodes, blob, B, "tiny", "exact", "amm", False, False, 0, 512)
    assert r["ok"] and r["mismatched_rows"] == 0 and r["rows"] >= 512
    bad = out.copy()
    bad.view(np.uint32)[-1, 0] ^= 1                       # last row: always sampled
    r = bench.rank_parity(tA, torch.from_numpy(bad), tcodes, blob, B, "tiny", "exact", "amm",
                          False, False, 0, 512)
    assert not r["ok"] and r["mismatched_rows"] == 1
    bc = O.pack_codes(codes)
    bc[-2, 0] ^= 0x10
    r = bench.rank_parity(tA, tout, torch.from_numpy(bc), blob, B, "tiny", "exact", "encode",
                          False, False, 0, 512)
    assert not r["ok"] and r["mismatched_rows"] == 1

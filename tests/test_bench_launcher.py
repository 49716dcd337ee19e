"""bench.py's multi-GPU launcher on CPU: --gpus 2 without torchrun re-executes
itself under torch.distributed.run with 2 ranks (127.0.0.1); the reference
arm (no CUDA) then runs on rank 0 only and prints one JSON line; and the
config-5 problem split gives every rank its contiguous share."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_gpus2_relaunches_under_torchrun_reference_arm():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # (rank 0 alone prints)
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                          "--impl", "reference"], capture_output=True, text=True, env=env,
                         timeout=120, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)


def test_config5_split_by_rank():
    sys.path.insert(0, ROOT)
    import bench
    os.environ["FINOM_BATCH"] = "10"
    try:
        parts = [bench.workload(5, r, 4) for r in range(4)]
    finally:
        os.environ.pop("FINOM_BATCH")
    sizes = [len(p["xs"]) for p in parts]
    assert sizes == [2, 3, 2, 3] and sum(sizes) == 10
    assert all(p["batch"] == 10 and p["itr"] == 200 for p in parts)

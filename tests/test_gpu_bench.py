"""bench.py contract on the GPU: one JSON line with the driver's keys, and the
multi-rank (torchrun) code path -- two ranks sharing device 0 over gloo, which
is only a smoke test of the launch / barrier / max-over-ranks plumbing."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c2", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--no-passes"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["value"] > 0
    assert d["gpu_launches"] > 0
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
        assert k in d["e2e"]["lazy"], k
    # the e2e step reads the four per-voxel output arrays back (the reference's output contract)
    assert d["e2e"]["d2h_bytes_per_step"] >= 17 * d["config"]["voxels"]
    assert "workload" in d["config"]


def test_reference_arm_same_config():
    """The reference arm prints the same `config` object as the B200 arm."""
    outs = []
    for extra in (["--impl", "reference", "--ref-budget", "5"], ["--no-cpu-baseline", "--no-passes", "--no-e2e"]):
        r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "2", "--warmup", "3"] + extra,
                           cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(_line(r.stdout))
    ref, ours = outs
    assert ref["impl"] == "reference" and ref["config"] == ours["config"]
    assert ref["metric"] == ours["metric"] and ref["unit"] == ours["unit"]


def test_bench_two_ranks_global_mode():
    """--gpus 2 in global mode (the driver's multi-GPU default): two processes
    share device 0 over gloo, each owns a z-slab, CUDA IPC peer reads, the
    calibration re-cut of the slab bounds gathered over the collective"""
    env = dict(os.environ, LRCVT_BENCH_DEVICE="0", LRCVT_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29563", "bench.py", "--gpus", "2",
                        "--config", "c2", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["mode"] == "global" and d["scaling"] == "strong" and d["value"] > 0
    assert len(d["slabs_z"]) == 2 and d["slabs_z"][0][0] == 0 and d["slabs_z"][1][1] == 128


def test_bench_two_ranks_smoke():
    env = dict(os.environ, LRCVT_BENCH_DEVICE="0", LRCVT_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "2",
                        "--config", "c2", "--mode", "blocks", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-passes", "--no-e2e"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0

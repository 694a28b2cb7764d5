"""The warp-per-voxel evaluation kernels (eval_warp.cuh) normally serve only
small frontiers (and the cooperative small-round kernel, default for 2D); LRCVT_WARP_EVAL=2 routes EVERY round through them, so the
reference-pinned classify tests (golden cases, fresh volumes vs the oracle,
20-iteration Lloyd trajectories) exercise their strict-order rule and exact
fallback on millions of evaluations. LRCVT_WARP_EVAL=0 checks the tile
kernels alone the same way."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("mode", ["2", "0", "coop", "ifchain"])
def test_classify_suite_under_forced_kernel_choice(mode):
    """mode "coop": every small frontier of every config goes through the
    persistent cooperative round kernel (rounds_small.cuh); mode "ifchain":
    the round graph selects the size class with one IF node per class
    instead of the SWITCH node (LRCVT_SWITCH=0)."""
    if mode == "coop":
        env = dict(os.environ, LRCVT_COOP="1")
    elif mode == "ifchain":
        env = dict(os.environ, LRCVT_SWITCH="0")
    else:
        env = dict(os.environ, LRCVT_WARP_EVAL=mode, LRCVT_COOP="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        str(ROOT / "tests" / "test_gpu_classify.py"), str(ROOT / "tests" / "test_gpu_edges.py"),
                        str(ROOT / "tests" / "test_gpu_blocks.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]

"""Time the one-off passes (masks, aggregation) on a config, per kernel under
ncu or by CUDA events: python tools/pass_bench.py [c3]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    import torch
    from paper_2208_06970_b200 import LloydParams, lrcvt
    from paper_2208_06970_b200.tessellation import engine_for

    grid, labels, params, sites, weights = bench.build_workload(bench.CONFIGS[cfg], 0)
    eng = engine_for(labels, grid.spacing, len(sites))
    tess, _ = lrcvt(grid, labels, params, LloydParams(max_updates=1))
    eng.ss[:, 0].copy_(torch.from_numpy(tess.site_of).cuda())
    t0 = time.perf_counter()
    out = bench.one_off_passes(grid, labels, eng, cfg, len(sites), reps=2)
    print(cfg, out, f"{time.perf_counter() - t0:.2f}s")


if __name__ == "__main__":
    main()

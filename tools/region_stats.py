"""Region shape statistics after a few Lloyd iterations (sizes and bounding
boxes of site_of regions): how much a per-site bounding-box scan would read
relative to the region sizes, and the worst site. Developer probe.

  python tools/region_stats.py --config c4
"""

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    cfg = bench.CONFIGS[a.config]
    grid, labels, params, sites, weights = bench.build_workload(cfg, 0)
    S = len(sites)
    eng = engine_for(labels, grid.spacing, S)
    pos = torch.from_numpy(np.array([s.position for s in sites])).cuda()
    sc = torch.from_numpy(np.array([s.component_id for s in sites], np.int32)).cuda()
    mode, w_d = lloyd_weight_mode(torch, grid, params, weights)
    vlen = voxel_length(grid.dims, grid.spacing)
    for _ in range(a.iters):
        eng.classify(pos, sc, want_state=False)
        pos, _, _, _ = eng.centroidal(pos, sc, mode, w_d, 0.5 * vlen)
    eng.classify(pos, sc, want_state=False)
    nx, ny, nz = grid.dims
    site = eng.ss[:, 0].long()
    m = site >= 0
    v = torch.nonzero(m).squeeze(1)
    s = site[v]
    x, y, z = v % nx, (v // nx) % ny, v // (nx * ny)
    cnt = torch.bincount(s, minlength=S).double()
    out = {}
    for name, c in (("x", x), ("y", y), ("z", z)):
        lo = torch.full((S,), 1 << 30, dtype=torch.long, device="cuda").scatter_reduce(0, s, c, "amin")
        hi = torch.full((S,), -1, dtype=torch.long, device="cuda").scatter_reduce(0, s, c, "amax")
        out[name] = (hi - lo + 1).clamp(min=0).double()
    box = out["x"] * out["y"] * out["z"]
    ratio = box / cnt.clamp(min=1)
    rows = out["y"] * out["z"]
    print(f"{a.config}: sites {S}, assigned {int(cnt.sum())}, sum bbox {float(box.sum()):.4g} "
          f"({float(box.sum() / cnt.sum()):.2f} x assigned)")
    for q in (0.5, 0.9, 0.99, 1.0):
        print(f"  q{q}: region {float(cnt.quantile(q)):.0f} bbox {float(box.quantile(q)):.0f} "
              f"ratio {float(ratio.quantile(q)):.2f} rows {float(rows.quantile(q)):.0f} xext {float(out['x'].quantile(q)):.0f}")
    i = int(torch.argmax(box))
    print(f"  worst site {i}: region {int(cnt[i])} bbox {int(box[i])} ext {int(out['x'][i])}x{int(out['y'][i])}x{int(out['z'][i])}")


if __name__ == "__main__":
    main()

"""One pass of every hot-path kernel inside an NVTX range named "profile",
for ncu (`--nvtx --nvtx-include "profile/"`): isobands + CCL + component
table, one Lloyd iteration (classify + vote + move) and the per-cell
aggregation (3 pairs + 64-bin histograms of f and g), after a warm-up of the
same calls. Same workload as bench.py --config <c>.

  python tools/profile_kernels.py --config c4
"""

from __future__ import annotations

import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--host-rounds", action="store_true",
                    help="host-driven relaxation rounds (plain launches instead of the conditional round graph, "
                         "whose kernel nodes ncu cannot profile individually)")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.pipeline import cell_aggregates_device
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    cfg = bench.CONFIGS[a.config]
    grid, labels, params, sites, weights = bench.build_workload(cfg, 0)
    L = _lib.lib()
    st = _lib.stream_handle(torch)
    n = grid.size
    nx, ny, nz = grid.dims
    S = len(sites)
    eng = engine_for(labels, grid.spacing, S)
    pos = torch.from_numpy(np.array([s.position for s in sites])).cuda()
    sc = torch.from_numpy(np.array([s.component_id for s in sites], np.int32)).cuda()
    mode, w_d = lloyd_weight_mode(torch, grid, params, weights)
    backoff = 0.5 * voxel_length(grid.dims, grid.spacing)
    f = torch.from_numpy(grid.fields["f"]).cuda()
    g = torch.from_numpy(grid.fields["g"]).cuda()
    iso = torch.tensor(cfg["iso"], dtype=torch.float64, device="cuda")
    layer = torch.empty(n, dtype=torch.int32, device="cuda")
    comp = torch.empty(n, dtype=torch.int32, device="cuda")
    ncomp = ctypes.c_int32()
    count = torch.empty(max(labels.n_components, 1), dtype=torch.int64, device="cuda")
    bbox = torch.empty((max(labels.n_components, 1), 6), dtype=torch.int32, device="cuda")
    lay = torch.empty(max(labels.n_components, 1), dtype=torch.int32, device="cuda")
    pairs = np.array([[0, 0], [0, 1], [1, 1]], np.int32)
    L.lrcvt_plan_reuse_eligible(eng.plan, 2)
    if a.host_rounds:
        _lib.check(L.lrcvt_plan_set_timing(eng.plan, 1), "set_timing")

    def once(p):
        _lib.check(L.lrcvt_isobands(n, f.data_ptr(), iso.data_ptr(), iso.numel(), layer.data_ptr(), st), "iso")
        _lib.check(L.lrcvt_label_components(nx, ny, nz, layer.data_ptr(), iso.numel() - 1, comp.data_ptr(),
                                            ctypes.byref(ncomp), st), "ccl")
        _lib.check(L.lrcvt_component_table(nx, ny, nz, comp.data_ptr(), layer.data_ptr(), ncomp.value,
                                           count.data_ptr(), bbox.data_ptr(), lay.data_ptr(), st), "table")
        eng.classify(p, sc, want_state=True)
        p2, _, _, _ = eng.centroidal(p, sc, mode, w_d, backoff)
        cell_aggregates_device([f, g], eng.comp, eng.ss[:, 0].contiguous(), S, labels.n_components, pairs, bins=64)
        return p2

    for _ in range(a.warm):
        pos = once(pos)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profile")
    pos = once(pos)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("profile pass done:", a.config, "sites", S, "rounds", eng.stats.rounds, "E", eng.stats.evaluations)


if __name__ == "__main__":
    main()

"""Aggregation pass probe at a bench config (python tools/agg_probe.py c4):
builds the workload, one Lloyd iteration for site_of, then times
cell_aggregates_device; run under ncu -k for the per-kernel split."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import numpy as np
    import torch

    from paper_2208_06970_b200.pipeline import cell_aggregates_device
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    grid, labels, params, sites, weights = bench.build_workload(bench.CONFIGS[cfg], 0)
    S = len(sites)
    eng = engine_for(labels, grid.spacing, S)
    pos = torch.from_numpy(np.array([s.position for s in sites])).cuda()
    sc = torch.from_numpy(np.array([s.component_id for s in sites], np.int32)).cuda()
    eng.classify(pos, sc)
    f = torch.from_numpy(grid.fields["f"]).cuda()
    g = torch.from_numpy(grid.fields["g"]).cuda()
    site_of = eng.ss[:, 0].contiguous()
    pairs = np.array([[0, 0], [0, 1], [1, 1]], np.int32)
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cell_aggregates_device([f, g], eng.comp, site_of, S, labels.n_components, pairs, bins=64)
        e1.record()
        torch.cuda.synchronize()
        print(f"rep {r}: aggregate {e0.elapsed_time(e1):.3f} ms", flush=True)


if __name__ == "__main__":
    main()

"""Where does the public-API step spend its time? (voronoi_classify + centroidal_update)"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch
    from paper_2208_06970_b200 import centroidal_update, voronoi_classify

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    grid, labels, params, sites, weights = bench.build_workload(bench.CONFIGS[cfg], 0)
    w = weights if params.weight_field else None
    for it in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tess = voronoi_classify(grid, labels, sites, w)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sites, ds = centroidal_update(tess)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"iter {it}: classify {1e3*(t1-t0):.2f} ms, update {1e3*(t2-t1):.2f} ms")
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        tess = voronoi_classify(grid, labels, sites, w)
        sites, ds = centroidal_update(tess)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()

"""Split the public-API update step: device call (synchronised) vs Python.

  python tools/e2e_probe2.py [c2|c4]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    from paper_2208_06970_b200 import centroidal_update, voronoi_classify
    from paper_2208_06970_b200 import tessellation as T

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    grid, labels, params, sites, weights = bench.build_workload(bench.CONFIGS[cfg], 0)
    acc = {"classify_dev": 0.0, "centroidal_dev": 0.0}
    orig_c, orig_u = T.Engine.classify, T.Engine.centroidal

    def wrap(name, fn):
        def inner(self, *a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn(self, *a, **k)
            torch.cuda.synchronize()
            acc[name] += time.perf_counter() - t0
            return r
        return inner

    T.Engine.classify = wrap("classify_dev", orig_c)
    T.Engine.centroidal = wrap("centroidal_dev", orig_u)
    w = weights
    for it in range(3):
        t = voronoi_classify(grid, labels, sites, w)
        sites, _ = centroidal_update(t)
    for k in acc:
        acc[k] = 0.0
    tc = tu = 0.0
    K = 10
    for it in range(K):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = voronoi_classify(grid, labels, sites, w)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sites, _ = centroidal_update(t)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        tc += t1 - t0
        tu += t2 - t1
    print(f"classify api {1e3 * tc / K:.3f} ms (engine {1e3 * acc['classify_dev'] / K:.3f}); "
          f"update api {1e3 * tu / K:.3f} ms (engine {1e3 * acc['centroidal_dev'] / K:.3f})")


if __name__ == "__main__":
    main()

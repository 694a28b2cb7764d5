import sys, cProfile, pstats
sys.path.insert(0, '.')
import bench
import torch
from paper_2208_06970_b200 import centroidal_update, voronoi_classify
grid, labels, params, sites, weights = bench.build_workload(bench.CONFIGS["c2"], 0)
for _ in range(3):
    t = voronoi_classify(grid, labels, sites, weights); sites, _ = centroidal_update(t)
torch.cuda.synchronize()
pr = cProfile.Profile()
for _ in range(20):
    t = voronoi_classify(grid, labels, sites, weights)
    torch.cuda.synchronize()
    pr.enable()
    sites, _ = centroidal_update(t)
    torch.cuda.synchronize()
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)

"""Global z-slab mode vs one domain on a bench workload, iteration by iteration
(GPU): the emulated K-slab GlobalClassifier and a single-domain Engine run the
same Lloyd iterations from the same sites; prints the first difference in the
classify counters, the per-voxel state of every slab, or the moved sites.

  python tools/mg_check.py [--config c4] [--ranks 8] [--iters 4] [--repeat 2]
"""

import argparse
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--uniform", action="store_true", help="equal-height slabs instead of balanced ones")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.multigpu import Emulated, GlobalClassifier
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    cfg = bench.CONFIGS[args.config]
    grid, labels, params, sites, weights = bench.build_workload(cfg, 0)
    S = len(sites)
    pos0 = torch.from_numpy(np.array([s.position for s in sites])).cuda()
    sc = torch.from_numpy(np.array([s.component_id for s in sites], np.int32)).cuda()
    mode, w_d = lloyd_weight_mode(torch, grid, params, weights)
    backoff = 0.5 * voxel_length(grid.dims, grid.spacing)
    L = _lib.lib()
    eng = engine_for(labels, grid.spacing, S)
    L.lrcvt_plan_reuse_eligible(eng.plan, 2)
    kw = {}
    if args.uniform:
        from paper_2208_06970_b200.multigpu import slab_bounds
        kw["bounds"] = slab_bounds(grid.dims[2], args.ranks)
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, S, Emulated(args.ranks),
                          **kw)
    if hasattr(gc, "reuse_sites"):
        gc.reuse_sites(True)
    print("slabs", gc.bounds, flush=True)
    p1, p2 = pos0.clone(), pos0.clone()
    ok = True
    for it in range(args.iters):
        st1 = eng.classify(p1, sc, want_state=True)
        st2 = gc.classify(p2, sc)
        c1 = {k: st1.get(k) for k in ("rounds", "sweeps", "evaluations", "commits", "assigned")}
        c2 = {k: st2.get(k) for k in ("rounds", "sweeps", "evaluations", "commits", "assigned")}
        same = True
        for r in gc.engines:
            v0, v1, e = gc.own_slab(r)
            for name in ("ss", "dist", "state"):
                a = getattr(eng, name)[v0:v1]
                b = getattr(e, name)[v0:v1]
                if not torch.equal(a, b):
                    nd = int((a != b).reshape(a.shape[0], -1).any(dim=1).sum())
                    print(f"iter {it} rank {r} {name}: {nd} voxels differ", flush=True)
                    same = False
        n1, _, _, _ = eng.centroidal(p1, sc, mode, w_d, backoff)
        n2, _, _ = gc.centroidal(p2, sc, mode, w_d, backoff)
        moved = torch.equal(n1, n2)
        h = hashlib.sha256(n2.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"iter {it}: single {c1}\n        global {c2}\n        state equal {same}, sites equal {moved}, "
              f"sha(global sites) {h}", flush=True)
        ok = ok and same and moved and c1["evaluations"] == c2["evaluations"]
        p1, p2 = n1, n2
    print("MG_CHECK", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

"""Global (z-slab) multi-GPU mode, emulated on one GPU: every rank's
replicated state and the report counters are bit-identical to the
single-domain classification, for 1-4 slabs; the full Lloyd trajectory in
global mode equals lrcvt()."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(kind, dims, iso, alpha, wf=None):
    from paper_2208_06970_b200 import (IsobandSpec, SeedingParams, classify_isobands, label_components,
                                       seed_sites, synth_field)

    grid = synth_field(kind, dims, 2)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", iso)))
    params = SeedingParams(alpha=alpha, seed=5, weight_field=wf)
    sites, _ = seed_sites(grid, labels, params)
    return grid, labels, params, sites


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("case", [("gaussian-mix", (40, 36, 48), [0.3, 0.7], 60),
                                  ("spiral", (44, 40, 37), [0.55, 0.75, 0.95], 80),
                                  ("horseshoe", (48, 48, 40), [0.0, 0.12, 0.3], 50)])
def test_global_classify_matches_single_domain(world, case):
    import torch

    from paper_2208_06970_b200 import voronoi_classify
    from paper_2208_06970_b200.multigpu import Emulated, GlobalClassifier

    grid, labels, params, sites = _setup(*case)
    ref = voronoi_classify(grid, labels, sites)
    pos = torch.from_numpy(ref.site_positions()).cuda()
    sc = torch.from_numpy(ref.site_components()).cuda()
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, len(sites),
                          Emulated(world))
    st = gc.classify(pos, sc)
    assert st["rounds"] == ref.report["rounds"] and st["sweeps"] == ref.report["sweeps"]
    assert st["assigned"] == ref.report["assigned"]
    assert st["evaluations"] == ref._b200_stats["evaluations"]
    assert st["commits"] == ref._b200_stats["commits"]
    for r in gc.engines:  # every rank's own slab
        v0, v1, eng = gc.own_slab(r)
        ss = eng.ss[v0:v1].cpu().numpy()
        assert np.array_equal(ss[:, 0], ref.site_of[v0:v1]), r
        assert np.array_equal(ss[:, 1], ref.src[v0:v1]), r
        assert np.array_equal(eng.dist[v0:v1].cpu().numpy(), ref.dist[v0:v1]), r
        assert np.array_equal(eng.state[v0:v1].cpu().numpy(), ref.state[v0:v1]), r


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("wf,gamma", [(None, 1.0), ("g", 1.0), ("g", 0.5)])
def test_global_centroidal_matches_single_domain(world, wf, gamma):
    """The slab-partitioned vote (integer all-reduce for unit weights, the
    running-sum hand-over for voxel-order fp64 chains) and the replicated
    move give the single-domain sums and sites bit for bit."""
    import torch

    from paper_2208_06970_b200 import SeedingParams, centroidal_update, seed_sites, voronoi_classify, voxel_weights
    from paper_2208_06970_b200.multigpu import Emulated, GlobalClassifier
    from paper_2208_06970_b200.tessellation import lloyd_weight_mode, voxel_length

    grid, labels, _, _ = _setup("random-smooth", (36, 40, 44), [0.35, 0.6, 0.8], 40)
    params = SeedingParams(alpha=70, seed=3, weight_field=wf, gamma=gamma)
    sites, _ = seed_sites(grid, labels, params)
    w = voxel_weights(grid, params)
    ref = voronoi_classify(grid, labels, sites, w)
    want, want_ds = centroidal_update(ref)
    pos = torch.from_numpy(ref.site_positions()).cuda()
    sc = torch.from_numpy(ref.site_components()).cuda()
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, len(sites),
                          Emulated(world))
    gc.classify(pos, sc)
    mode, w_d = lloyd_weight_mode(torch, grid, params, w)
    vlen = voxel_length(grid.dims, grid.spacing)
    new_pos, disp, _ = gc.centroidal(pos, sc, mode, w_d, 0.5 * vlen)
    assert np.array_equal(new_pos.cpu().numpy(), np.array([s.position for s in want]))
    assert float(disp.cpu().numpy().mean() / vlen) == want_ds


@pytest.mark.parametrize("world", [2, 4])
def test_global_lloyd_matches_lrcvt(world):
    from paper_2208_06970_b200 import LloydParams, lrcvt
    from paper_2208_06970_b200.multigpu import Emulated, global_lrcvt

    grid, labels, params, sites = _setup("gaussian-mix", (40, 40, 40), [0.3, 0.7], 70, wf="g")
    lp = LloydParams(max_updates=4, ds_tolerance=1e-9)
    ref, tr = lrcvt(grid, labels, params, lp)
    got, tg = global_lrcvt(grid, labels, params, lp, Emulated(world))
    assert tg == tr
    for k in ("site_of", "dist", "src", "state"):
        assert np.array_equal(getattr(got, k), getattr(ref, k)), k
    assert np.array_equal(got.site_positions(), ref.site_positions())


def test_global_classify_over_nccl_single_rank():
    """The torch.distributed (NCCL) collective path end to end on one rank."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2208_06970_b200 import voronoi_classify
    from paper_2208_06970_b200.multigpu import GlobalClassifier, TorchDist

    grid, labels, params, sites = _setup("gaussian-mix", (40, 36, 48), [0.3, 0.7], 60)
    ref = voronoi_classify(grid, labels, sites)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, len(sites),
                              TorchDist())
        st = gc.classify(torch.from_numpy(ref.site_positions()).cuda(),
                         torch.from_numpy(ref.site_components()).cuda())
        eng = gc.any_engine()
        assert np.array_equal(eng.ss.cpu().numpy()[:, 0], ref.site_of)
        assert np.array_equal(eng.dist.cpu().numpy(), ref.dist)
        assert np.array_equal(eng.state.cpu().numpy(), ref.state)
        assert st["evaluations"] == ref._b200_stats["evaluations"]
    finally:
        dist.destroy_process_group()


def _two_proc_worker(rank, world, port, outdir):
    """One rank per process, both on cuda:0: gloo (host) for the collectives,
    CUDA IPC mappings of the other rank's state buffers for the far reads."""
    import os
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    from paper_2208_06970_b200 import SeedingParams, centroidal_update, seed_sites, voronoi_classify, voxel_weights
    from paper_2208_06970_b200.multigpu import GlobalClassifier, TorchDist
    from paper_2208_06970_b200.tessellation import lloyd_weight_mode, voxel_length

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, labels, _, _ = _setup("horseshoe", (48, 44, 40), [0.0, 0.12, 0.3], 50)
        params = SeedingParams(alpha=60, seed=5, weight_field="g")
        sites, _ = seed_sites(grid, labels, params)
        w = voxel_weights(grid, params)
        ref = voronoi_classify(grid, labels, sites, w)
        want, _ = centroidal_update(ref)
        pos = torch.from_numpy(ref.site_positions()).cuda()
        sc = torch.from_numpy(ref.site_components()).cuda()
        coll = TorchDist(device="cpu")
        gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, len(sites), coll)
        st = gc.classify(pos, sc)
        v0, v1, eng = gc.own_slab(rank)
        ok = (np.array_equal(eng.ss[v0:v1].cpu().numpy()[:, 0], ref.site_of[v0:v1])
              and np.array_equal(eng.ss[v0:v1].cpu().numpy()[:, 1], ref.src[v0:v1])
              and np.array_equal(eng.dist[v0:v1].cpu().numpy(), ref.dist[v0:v1])
              and np.array_equal(eng.state[v0:v1].cpu().numpy(), ref.state[v0:v1])
              and st["rounds"] == ref.report["rounds"] and st["sweeps"] == ref.report["sweeps"]
              and st["evaluations"] == ref._b200_stats["evaluations"] and st["assigned"] == ref.report["assigned"])
        mode, w_d = lloyd_weight_mode(torch, grid, params, w)
        new_pos, _, _ = gc.centroidal(pos, sc, mode, w_d, 0.5 * voxel_length(grid.dims, grid.spacing))
        ok = ok and np.array_equal(new_pos.cpu().numpy(), np.array([s.position for s in want]))
        torch.cuda.synchronize()
        dist.barrier()
        coll.close()
        Path(outdir, f"r{rank}").write_text("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


def test_global_classify_two_processes_gloo_ipc():
    """2 processes x 1 shared GPU: the TorchDist protocol (gloo, host-staged)
    with CUDA-IPC peer reads gives the single-domain result on both slabs."""
    import os
    import socket
    import tempfile

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_two_proc_worker, args=(2, port, d), nprocs=2, join=True)
        for r in range(2):
            assert open(os.path.join(d, f"r{r}")).read() == "ok", r


@pytest.mark.parametrize("world", [2, 3])
def test_global_lloyd_large_frontiers_matches_single_domain(world):
    """Frontiers of tens of thousands of voxels per slab (the thread-per-voxel
    eval kernels, not only the warp-per-voxel ones), balanced slabs, the
    eligible list kept across Lloyd iterations, slabs re-cut before the third:
    arrays, counters and the moved sites equal the single-domain engine's."""
    import torch

    from paper_2208_06970_b200 import SeedingParams, seed_sites, voxel_weights
    from paper_2208_06970_b200.multigpu import Emulated, GlobalClassifier
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    grid, labels, _, _ = _setup("random-smooth", (96, 88, 80), [0.35, 0.5, 0.65], 40)
    params = SeedingParams(alpha=600, seed=7, weight_field="g", gamma=1.0)
    sites, _ = seed_sites(grid, labels, params)
    w = voxel_weights(grid, params)
    S = len(sites)
    pos = torch.from_numpy(np.array([s.position for s in sites])).cuda()
    sc = torch.from_numpy(np.array([s.component_id for s in sites], np.int32)).cuda()
    mode, w_d = lloyd_weight_mode(torch, grid, params, w)
    backoff = 0.5 * voxel_length(grid.dims, grid.spacing)
    eng = engine_for(labels, grid.spacing, S)
    eng.L.lrcvt_plan_reuse_eligible(eng.plan, 2)
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, S, Emulated(world))
    gc.reuse_sites(True)
    p1, p2 = pos.clone(), pos.clone()
    try:
        for it in range(3):
            if it == 2:  # re-cut the slabs mid-run (rebalance from made-up costs): still bit-identical
                old = list(gc.bounds)
                assert gc.rebalance({r: 3.0 if r == 0 else 1.0 for r in gc.engines}) != old
            st1 = eng.classify(p1, sc, want_state=True)
            st2 = gc.classify(p2, sc)
            assert st1["evaluations"] > 2048 * world * 10
            for k in ("rounds", "sweeps", "evaluations", "commits", "assigned"):
                assert st1[k] == st2[k], k
            for r in gc.engines:
                v0, v1, e = gc.own_slab(r)
                for name in ("ss", "dist", "state"):
                    assert torch.equal(getattr(eng, name)[v0:v1], getattr(e, name)[v0:v1]), (r, name)
            p1, _, _, _ = eng.centroidal(p1, sc, mode, w_d, backoff)
            p2, _, _ = gc.centroidal(p2, sc, mode, w_d, backoff)
            assert torch.equal(p1, p2)
    finally:
        eng.L.lrcvt_plan_reuse_eligible(eng.plan, 0)

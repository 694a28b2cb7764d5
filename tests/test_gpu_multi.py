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
    for r, eng in gc.engines.items():
        ss = eng.ss.cpu().numpy()
        assert np.array_equal(ss[:, 0], ref.site_of), r
        assert np.array_equal(ss[:, 1], ref.src), r
        assert np.array_equal(eng.dist.cpu().numpy(), ref.dist), r
        assert np.array_equal(eng.state.cpu().numpy(), ref.state), r


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
        assert st["evaluations"] == ref._b200_stats["evaluations"]
    finally:
        dist.destroy_process_group()

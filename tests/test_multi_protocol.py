"""CPU (gloo, world_size 2): the global-mode collective protocol -- count
exchange and rank-ordered proposal concatenation with unequal and zero
sizes -- plus slab partitioning."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def test_slab_bounds():
    from paper_2208_06970_b200.multigpu import slab_bounds

    assert slab_bounds(128, 1) == [(0, 128)]
    assert slab_bounds(128, 3) == [(0, 43), (43, 86), (86, 128)]
    assert slab_bounds(1024, 8)[-1] == (896, 1024)
    b = slab_bounds(37, 4)
    assert b[0][0] == 0 and b[-1][1] == 37 and all(lo < hi for lo, hi in b)
    with pytest.raises(ValueError):
        slab_bounds(3, 4)


def _worker(rank, world, port, outdir):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from paper_2208_06970_b200.multigpu import PROP_BYTES, TorchDist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coll = TorchDist(device="cpu")
        assert coll.local_ranks == [rank] and coll.world == world
        assert coll.all_counts([rank * 10 + 1]) == [r * 10 + 1 for r in range(world)]
        for sizes in ([3, 5], [0, 4], [0, 0], [7, 0]):
            mine = sizes[rank] * PROP_BYTES
            local = torch.arange(mine, dtype=torch.int64).remainder(251).to(torch.uint8) + rank
            got = coll.all_props([local], torch)
            want = torch.cat([torch.arange(s * PROP_BYTES, dtype=torch.int64).remainder(251).to(torch.uint8) + r
                              for r, s in enumerate(sizes)])
            assert torch.equal(got, want), sizes
        Path(outdir, f"ok{rank}").write_text("ok")
    finally:
        dist.destroy_process_group()


def test_collective_protocol_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, port, d), nprocs=2, join=True)
        assert os.path.exists(os.path.join(d, "ok0")) and os.path.exists(os.path.join(d, "ok1"))

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


def test_cost_balanced_bounds():
    """measured per-rank costs move the cuts toward the expensive slab; equal
    intensities keep the in-band balance"""
    from paper_2208_06970_b200.multigpu import cost_balanced_bounds, plane_inband

    inb = np.ones(100)
    b = [(0, 25), (25, 50), (50, 75), (75, 100)]
    assert cost_balanced_bounds(inb, b, [1, 1, 1, 1]) == b
    nb = cost_balanced_bounds(inb, b, [2, 1, 1, 1])
    assert nb[0][1] < 25 and nb[0][0] == 0 and nb[-1][1] == 100
    assert all(lo < hi for lo, hi in nb) and all(nb[r][1] == nb[r + 1][0] for r in range(3))
    comp = np.full((6, 4, 4), -1, np.int32)
    comp[:, :, :2] = 0
    assert plane_inband(comp.reshape(-1), (4, 4, 6)).tolist() == [8.0] * 6


class _CpuTorch:
    """torch with "cuda" tensors mapped to the CPU (the protocol test has no GPU)."""

    def __getattr__(self, name):
        return getattr(torch, name)

    @staticmethod
    def empty(*a, device=None, **k):
        return torch.empty(*a, **k)

    @staticmethod
    def cat(ts):
        return torch.cat(ts)


_CpuTorch = _CpuTorch()


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
        assert coll.gather_floats({rank: 0.5 + rank}) == [0.5 + r for r in range(world)]  # rebalance costs
        for sizes in ([3, 5], [0, 4], [0, 0], [7, 0]):
            mine = sizes[rank] * PROP_BYTES
            local = torch.arange(mine, dtype=torch.int64).remainder(251).to(torch.uint8) + rank
            got = coll.all_props([local], torch)
            want = torch.cat([torch.arange(s * PROP_BYTES, dtype=torch.int64).remainder(251).to(torch.uint8) + r
                              for r, s in enumerate(sizes)])
            assert torch.equal(got, want), sizes
        # halo exchange: rank r receives hi of r - 1 and lo of r + 1
        lo = {rank: torch.full((rank * 24,), 10 + rank, dtype=torch.uint8)}
        hi = {rank: torch.full((24 + rank * 48,), 20 + rank, dtype=torch.uint8)}
        got = coll.exchange_halo(lo, hi, _CpuTorch)[rank]
        want = []
        if rank > 0:
            want.append(torch.full((24 + (rank - 1) * 48,), 20 + rank - 1, dtype=torch.uint8))
        if rank + 1 < world:
            want.append(torch.full(((rank + 1) * 24,), 10 + rank + 1, dtype=torch.uint8))
        want = torch.cat(want) if want else torch.empty(0, dtype=torch.uint8)
        assert torch.equal(got.cpu(), want)
        # all-reduce ops and the rank-ordered carry chain (the ordered vote hand-over)
        t = torch.tensor([[rank + 1, -rank], [5 * rank, 7]], dtype=torch.int64)
        assert torch.equal(coll.allreduce({rank: t}, "sum", _CpuTorch).cpu(),
                           sum(torch.tensor([[r + 1, -r], [5 * r, 7]]) for r in range(world)))
        assert torch.equal(coll.allreduce({rank: t}, "min", _CpuTorch).cpu(), torch.tensor([[1, -(world - 1)], [0, 7]]))
        assert torch.equal(coll.allreduce({rank: t}, "max", _CpuTorch).cpu(),
                           torch.tensor([[world, 0], [5 * (world - 1), 7]]))

        def step(r, carry):
            # non-associative on purpose: the order of the hand-over matters
            base = torch.zeros((4, 3), dtype=torch.float64) if carry is None else carry.cpu()
            return base * 0.5 + (r + 1)

        final = coll.chain(step, (4, 3), _CpuTorch).cpu()
        want_c = torch.zeros((4, 3), dtype=torch.float64)
        for r in range(world):
            want_c = want_c * 0.5 + (r + 1)
        assert torch.equal(final, want_c)
        assert coll.sum_ints({rank: [rank, 1]}) == [sum(range(world)), world]
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


def test_balanced_slab_bounds():
    from paper_2208_06970_b200.multigpu import balanced_slab_bounds

    nx, ny, nz = 4, 3, 40
    comp = -np.ones((nz, ny, nx), np.int32)
    comp[30:] = 0  # all in-band voxels in the top 10 planes
    b = balanced_slab_bounds(comp.ravel(), (nx, ny, nz), 4)
    assert b[0][0] == 0 and b[-1][1] == nz and all(lo < hi for lo, hi in b)
    assert all(b[i][1] == b[i + 1][0] for i in range(3))
    counts = [int(np.count_nonzero(comp[lo:hi] >= 0)) for lo, hi in b]
    assert max(counts) - min(counts) <= ny * nx * 2  # balanced to within a couple of planes
    assert balanced_slab_bounds(np.zeros(nx * ny * nz, np.int32), (nx, ny, nz), 40) == [(z, z + 1) for z in range(40)]

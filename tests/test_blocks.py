"""Block mode (the reference's distributed semantics, pipeline.py:45-160):
the sequential driver and the torch.distributed driver (world_size 2, gloo,
CPU) against block-mode golden vectors from the reference. Per-block compute
is the CPU oracle here; the GPU variants are in test_gpu_blocks.py."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import case_arrays, load_json, load_npz

CASES = ["spiral48_b221", "smooth24_b112", "gmix20_b212"]


def _params(m):
    from paper_2208_06970_b200 import IsobandSpec, LloydParams, SeedingParams, synth_field

    return (synth_field(m["kind"], tuple(m["dims"]), 0), IsobandSpec("f", m["iso"]), SeedingParams(**m["seeding"]),
            LloydParams(**m["lloyd"]), tuple(m["blocks"]))


def check_result(res, m, a):
    for key in ("site_of", "dist", "src", "state"):
        assert np.array_equal(getattr(res.tess, key), a[key]), key
    assert np.array_equal(res.labels.layer, a["layer"])
    assert np.array_equal(res.labels.component, a["component"])
    got_sites = np.array([[*s.position, s.component_id] for s in res.tess.sites])
    assert np.array_equal(got_sites, a["sites"])
    assert res.trace == m["trace"]
    assert [list(t) for t in res.block_traces] == m["block_traces"]
    assert [(c.id, c.layer, c.voxel_count, list(c.bbox)) for c in res.labels.component_table] == \
           [(t["id"], t["layer"], t["voxel_count"], t["bbox"]) for t in m["table"]]


@pytest.mark.parametrize("case", CASES)
def test_sequential_block_mode_matches_reference(case, oracle_mod):
    from blockfns import oracle_label, oracle_lloyd
    from paper_2208_06970_b200.pipeline import run_pipeline

    m, a = load_json("blocks.json")[case], case_arrays(load_npz("blocks.npz"), case)
    grid, iso, sp, lp, blocks = _params(m)
    res = run_pipeline(grid, iso, sp, lp, blocks, label_fn=oracle_label, lloyd_fn=oracle_lloyd)
    check_result(res, m, a)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, outdir):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from blockfns import oracle_label, oracle_lloyd
    from conftest import case_arrays, load_json, load_npz
    from paper_2208_06970_b200.pipeline import run_pipeline_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, a = load_json("blocks.json")[case], case_arrays(load_npz("blocks.npz"), case)
        grid, iso, sp, lp, blocks = _params(m)
        res = run_pipeline_distributed(grid, iso, sp, lp, blocks, label_fn=oracle_label, lloyd_fn=oracle_lloyd)
        if rank == 0:
            check_result(res, m, a)
            Path(outdir, "ok").write_text("ok")
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES)
def test_distributed_block_mode_gloo_world2(case):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), case, d), nprocs=2, join=True)
        assert os.path.exists(os.path.join(d, "ok"))

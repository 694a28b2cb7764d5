"""GPU block mode: run_pipeline and the torch.distributed block driver
(single-rank group on cuda:0) against the reference's block-mode golden
vectors, bit-exact."""

import os
import socket

import numpy as np
import pytest

from conftest import case_arrays, load_json, load_npz
from test_blocks import CASES, _params, check_result

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", CASES)
def test_gpu_block_mode_matches_reference(case):
    from paper_2208_06970_b200.pipeline import run_pipeline

    m, a = load_json("blocks.json")[case], case_arrays(load_npz("blocks.npz"), case)
    grid, iso, sp, lp, blocks = _params(m)
    check_result(run_pipeline(grid, iso, sp, lp, blocks), m, a)


def test_gpu_distributed_driver_single_rank():
    import torch.distributed as dist

    from paper_2208_06970_b200.pipeline import run_pipeline_distributed

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        for case in CASES:
            m, a = load_json("blocks.json")[case], case_arrays(load_npz("blocks.npz"), case)
            grid, iso, sp, lp, blocks = _params(m)
            check_result(run_pipeline_distributed(grid, iso, sp, lp, blocks), m, a)
    finally:
        dist.destroy_process_group()

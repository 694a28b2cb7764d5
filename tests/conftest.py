import json
import gzip
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_npz(name):
    return np.load(GOLDEN / name, allow_pickle=False)


def load_json(name):
    p = GOLDEN / name
    if name.endswith(".gz"):
        with gzip.open(p, "rt") as fh:
            return json.load(fh)
    return json.loads(p.read_text())


def case_arrays(npz, name):
    pre = f"{name}/"
    return {k[len(pre):]: npz[k] for k in npz.files if k.startswith(pre)}


@pytest.fixture(scope="session")
def classify_golden():
    return load_npz("classify.npz"), load_json("classify.json")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle

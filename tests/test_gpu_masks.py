"""GPU parity: isoband classification and connected-component labelling
(ids, table) against the reference's golden vectors and the scipy oracle,
bit-exact."""

import numpy as np
import pytest

from conftest import case_arrays, load_json, load_npz

pytestmark = pytest.mark.gpu


def _grid_for(name, m, a):
    from paper_2208_06970_b200 import VoxelGrid, synth_field

    if "f" in a:
        return VoxelGrid(tuple(m["dims"]), (1, 1, 1), {"f": a["f"]})
    kinds = {"rings40": ("rings", 1), "spiral64": ("spiral", 0), "spiral48_3d": ("spiral", 0),
             "horseshoe64": ("horseshoe", 0), "smooth24": ("random-smooth", 3)}
    kind, seed = kinds[name]
    return synth_field(kind, tuple(m["dims"]), seed)


def test_masks_golden():
    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components

    npz, meta = load_npz("masks.npz"), load_json("masks.json.gz")
    for name, m in meta.items():
        a = case_arrays(npz, name)
        grid = _grid_for(name, m, a)
        lm = classify_isobands(grid, IsobandSpec("f", m["iso"]))
        assert np.array_equal(lm.layer, a["layer"]), name
        assert np.all(lm.component == -1)
        labels = label_components(lm)
        assert np.array_equal(labels.component, a["component"]), name
        got = [(c.id, c.layer, c.voxel_count, list(c.bbox), list(c.band)) for c in labels.component_table]
        want = [(t["id"], t["layer"], t["voxel_count"], t["bbox"], t["band"]) for t in m["table"]]
        assert got == want, name


@pytest.mark.parametrize("dims,seed", [((64, 64, 64), 0), ((200, 3, 70), 1), ((1000, 1, 1), 2),
                                       ((96, 80, 1), 3)])
def test_ccl_vs_oracle_random(dims, seed, oracle_mod):
    from paper_2208_06970_b200 import IsobandSpec, VoxelGrid, classify_isobands, label_components

    rng = np.random.default_rng(seed)
    f = rng.random(int(np.prod(dims))).astype(np.float32)
    grid = VoxelGrid(dims, (1, 1, 1), {"f": f})
    iso = [0.2, 0.45, 0.7, 0.95]
    labels = label_components(classify_isobands(grid, IsobandSpec("f", iso)))
    layer = oracle_mod.isobands(f, iso)
    assert np.array_equal(labels.layer, layer)
    comp, table = oracle_mod.label_components(layer, dims, len(iso) - 1)
    assert np.array_equal(labels.component, comp)
    assert [(c.id, c.layer, c.voxel_count, list(c.bbox)) for c in labels.component_table] == \
           [(t["id"], t["layer"], t["voxel_count"], t["bbox"]) for t in table]


def test_isoband_edges_exact():
    """Values exactly on iso values: lower edge out, upper edge in."""
    from paper_2208_06970_b200 import IsobandSpec, VoxelGrid, classify_isobands

    iso = [0.25, 0.5, 0.75]
    f = np.array([0.25, 0.5, 0.75, 0.2500001, np.nextafter(np.float32(0.75), 1), 0.0, 1.0], np.float32)
    lm = classify_isobands(VoxelGrid((7, 1, 1), (1, 1, 1), {"f": f}), IsobandSpec("f", iso))
    assert lm.layer.tolist() == [-1, 0, 1, 0, -1, -1, -1]

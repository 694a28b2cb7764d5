"""GPU seeding masses (lrcvt_seed_masses) against the
host numpy table (seeding.py:71-107 semantics) and the reference's golden
sites: every group's index, voxels, weights and mass, the per-component and
total masses, all bit-identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same_table(a, b):
    assert a.total_mass == b.total_mass
    assert a.comp_mass.tobytes() == b.comp_mass.tobytes()
    assert len(a.comp_blocks) == len(b.comp_blocks)
    for ba, bb in zip(a.comp_blocks, b.comp_blocks):
        assert [x.index for x in ba] == [x.index for x in bb]
        assert [x.mass for x in ba] == [x.mass for x in bb]
        for x, y in zip(ba, bb):
            assert np.array_equal(x.voxels, y.voxels)
            assert x.weights.tobytes() == y.weights.tobytes()


CASES = [
    ("spiral", (96, 80, 1), [0.3, 0.55, 0.8], "g", 1.0, 16),
    ("gaussian-mix", (48, 40, 36), [0.3, 0.7], "g", 1.0, 16),
    ("random-smooth", (40, 40, 40), [0.35, 0.5, 0.65, 0.8], "g", 2.0, 8),
    ("horseshoe", (48, 48, 48), [0.0, 0.12, 0.3], None, 1.0, 16),
    ("random-smooth", (33, 29, 31), [0.4, 0.6], "f", 0.5, 7),
    ("gaussian-mix", (64, 64, 64), [0.3, 0.7], "g", 1.0, 64),
    ("gaussian-mix", (20, 18, 16), [0.3, 0.7], "g", 1.0, 1),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[5]}-{c[4]}" for c in CASES])
def test_device_masses_equal_host(case):
    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components, synth_field
    from paper_2208_06970_b200.seeding import SeedingParams, component_masses, component_masses_device

    kind, dims, iso, wf, gamma, bs = case
    grid = synth_field(kind, dims, 0)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", iso)))
    params = SeedingParams(alpha=64, gamma=gamma, weight_field=wf, block_size=bs, seed=3)
    _same_table(component_masses_device(grid, labels, params), component_masses(grid, labels, params))


def test_device_seeding_matches_reference_golden():
    """seed_sites on the GPU table reproduces the reference's own sites."""
    import json
    from pathlib import Path

    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components, synth_field
    from paper_2208_06970_b200.seeding import SeedingParams, seed_sites

    gold = json.loads((Path(__file__).resolve().parent / "golden" / "seeding.json").read_text())

    for name, m in gold.items():
        g = synth_field(m["kind"], tuple(m["dims"]), 0)
        labels = label_components(classify_isobands(g, IsobandSpec("f", m["iso"])))
        sites, rep = seed_sites(g, labels, SeedingParams(**m["params"]), device=True)
        assert [[*s.position, s.component_id] for s in sites] == m["sites"], name
        assert rep["target_counts"] == m["report"]["target_counts"], name


def test_device_masses_dummy_table_retries():
    """A component table with understated bounding boxes still works."""
    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components, synth_field
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap
    from paper_2208_06970_b200.seeding import SeedingParams, component_masses, component_masses_device

    grid = synth_field("gaussian-mix", (40, 36, 32), 0)
    lab = label_components(classify_isobands(grid, IsobandSpec("f", [0.3, 0.7])))
    dummy = LabelMap(lab.dims, lab.layer, lab.component,
                     [ComponentInfo(c.id, c.layer, 1, (0,) * 6, c.band) for c in lab.component_table],
                     lab.iso_values, lab.field_name)
    params = SeedingParams(alpha=32, weight_field="g", block_size=8)
    _same_table(component_masses_device(grid, dummy, params), component_masses(grid, lab, params))


def test_device_masses_negative_weights_raise():
    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components, synth_field
    from paper_2208_06970_b200.seeding import SeedingParams, component_masses_device

    grid = synth_field("gaussian-mix", (16, 16, 16), 0)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.3, 0.7])))
    grid.fields["neg"] = (grid.fields["g"] - 0.5).astype(np.float32)
    with pytest.raises(ValueError, match="negative"):
        component_masses_device(grid, labels, SeedingParams(weight_field="neg"))
    with pytest.raises(KeyError):
        component_masses_device(grid, labels, SeedingParams(weight_field="nope"))

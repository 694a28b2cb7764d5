"""GPU parity: CUDA classification / centroid vote / site move / rays against
the reference's golden vectors and the CPU oracle, bit-exact.

Tolerance: none -- site_of, src, dist, state, report counters, vote sums and
new site positions must be bit-identical (fp64, no FMA contraction on either
side; unit-weight sums are exact integers, weighted sums are added in the
reference's voxel order)."""

import hashlib

import numpy as np
import pytest

from conftest import case_arrays, load_json, load_npz

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def labels_from_comp(dims, comp, n_components, layer=None):
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap

    comp = np.ascontiguousarray(comp, dtype=np.int32)
    if layer is None:
        layer = np.where(comp >= 0, 0, -1).astype(np.int32)
    counts = np.bincount(comp[comp >= 0], minlength=n_components)
    table = [ComponentInfo(c, 0, int(counts[c]), (0, 0, 0, 0, 0, 0), (0.0, 1.0)) for c in range(n_components)]
    return LabelMap(tuple(dims), layer, comp, table, [0.0, 1.0], "f")


def sites_of(pos, comp):
    from paper_2208_06970_b200.seeding import Site

    return [Site(tuple(float(t) for t in p), int(c)) for p, c in zip(pos, comp)]


def test_classify_golden_cases(classify_golden):
    from paper_2208_06970_b200 import VoxelGrid, voronoi_classify

    npz, meta = classify_golden
    for name, m in meta.items():
        a = case_arrays(npz, name)
        grid = VoxelGrid(tuple(m["dims"]), tuple(m["spacing"]), {})
        labels = labels_from_comp(m["dims"], a["comp"], m["n_components"])
        tess = voronoi_classify(grid, labels, sites_of(a["site_pos"], a["site_comp"]), a.get("weights"))
        for key in ("site_of", "dist", "src", "state"):
            assert np.array_equal(getattr(tess, key), a[key]), (name, key)
        rep = m["report"]
        assert tess.report["rounds"] == rep["rounds"], name
        assert tess.report["sweeps"] == rep["sweeps"], name
        assert tess.report["assigned"] == rep["assigned"], name
        assert tess.report["components_without_sites"] == rep["components_without_sites"], name


def test_centroidal_golden_cases(classify_golden):
    from paper_2208_06970_b200 import VoxelGrid, centroidal_update, voronoi_classify

    npz, meta = classify_golden
    for name, m in meta.items():
        a = case_arrays(npz, name)
        grid = VoxelGrid(tuple(m["dims"]), tuple(m["spacing"]), {})
        labels = labels_from_comp(m["dims"], a["comp"], m["n_components"])
        tess = voronoi_classify(grid, labels, sites_of(a["site_pos"], a["site_comp"]), a.get("weights"))
        new_sites, mean_ds = centroidal_update(tess)
        got = np.array([s.position for s in new_sites])
        assert np.array_equal(got, a["new_pos"]), name
        assert mean_ds == m["mean_ds"], name
        assert tess.report["empty_regions"] == m["empty_regions"], name


def test_centroid_sums_bit_exact_all_weight_modes(classify_golden):
    """Both vote paths (exact-integer for unit weights, ordered for f64
    weights) reproduce the reference's per-site sums bit for bit."""
    import torch

    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.tessellation import Engine

    npz, meta = classify_golden
    for name, m in meta.items():
        a = case_arrays(npz, name)
        eng = Engine(tuple(m["dims"]), tuple(m["spacing"]), a["comp"], m["n_components"], len(a["site_comp"]))
        eng.upload(a["site_of"], a["src"])
        pos = torch.from_numpy(a["site_pos"]).cuda()
        sc = torch.from_numpy(a["site_comp"]).cuda()
        w = a.get("weights")
        modes = [(_lib.W_F64, torch.from_numpy(np.ones(len(a["comp"])) if w is None else w).cuda())]
        if w is None:
            modes.append((_lib.W_ONES, None))
        for mode, wd in modes:
            _, _, _, sums = eng.centroidal(pos, sc, mode, wd, 0.5, want_sums=True)
            assert np.array_equal(sums.cpu().numpy(), a["sums4"]), (name, mode)


def test_site_outside_component_rejected():
    from paper_2208_06970_b200 import VoxelGrid, voronoi_classify
    from paper_2208_06970_b200.seeding import Site

    grid = VoxelGrid((8, 8, 1), (1, 1, 1), {})
    labels = labels_from_comp((8, 8, 1), np.zeros(64, np.int32), 1)
    with pytest.raises(ValueError, match="outside"):
        voronoi_classify(grid, labels, [Site((4.5, 4.5, 0.5), 3)])


def test_raycast_golden():
    from paper_2208_06970_b200.tessellation import raycast_same_component, segment_hit_t_batch

    npz, meta = load_npz("raycast.npz"), load_json("raycast.json")
    for name, m in meta.items():
        a = case_arrays(npz, name)
        labels = labels_from_comp(m["dims"], a["comp"], int(a["comp"].max()) + 1)
        t = segment_hit_t_batch(labels, a["segs"], a["want"], m["spacing"])
        assert np.array_equal(t, a["t"]), name
        s = a["segs"][0]
        assert raycast_same_component(labels, s[:3], s[3:], m["spacing"]) == bool(a["t"][0] >= 1.0)


@pytest.mark.parametrize("kind,dims,iso,alpha,wf,gamma", [
    ("random-smooth", (40, 36, 32), [0.35, 0.6, 0.8], 90, "g", 1.0),
    ("spiral", (128, 128, 1), [0.3, 0.55, 0.8], 120, None, 1.0),
    ("horseshoe", (48, 48, 48), [0.0, 0.12, 0.3], 70, "g", 0.5),
    ("gaussian-mix", (33, 29, 31), [0.3, 0.7], 50, "g", 2.0),
])
def test_classify_and_update_vs_oracle(kind, dims, iso, alpha, wf, gamma, oracle_mod):
    """Fresh seeded volumes (not in the golden set): CUDA vs oracle, with the
    E (evaluations) and C (commits) schedule counters equal too."""
    from paper_2208_06970_b200 import (IsobandSpec, SeedingParams, centroidal_update, classify_isobands,
                                       label_components, seed_sites, synth_field, voronoi_classify,
                                       voxel_weights)

    grid = synth_field(kind, dims, 3)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", iso)))
    params = SeedingParams(alpha=alpha, seed=11, weight_field=wf, gamma=gamma)
    sites, _ = seed_sites(grid, labels, params)
    w = voxel_weights(grid, params)
    tess = voronoi_classify(grid, labels, sites, w)
    pos = tess.site_positions()
    sc = tess.site_components()
    ref = oracle_mod.classify(dims, grid.spacing, labels.component, pos, sc, labels.n_components)
    for key in ("site_of", "dist", "src", "state"):
        assert np.array_equal(getattr(tess, key), ref[key]), key
    assert tess.report["rounds"] == ref["rounds"]
    assert tess.report["sweeps"] == ref["sweeps"]
    assert tess._b200_stats["evaluations"] == ref["evaluations"]
    assert tess._b200_stats["commits"] == ref["commits"]
    new_sites, mean_ds = centroidal_update(tess)
    u = oracle_mod.centroidal(dims, grid.spacing, labels.component, ref["site_of"], ref["src"], w, pos, sc)
    assert np.array_equal(np.array([s.position for s in new_sites]), u["new_pos"])
    assert mean_ds == u["mean_ds"]


@pytest.mark.parametrize("case", ["spiral48_det", "smooth32_3d_g2", "c1_spiral256", "c2_gmix128"])
def test_lloyd_trajectory_matches_reference(case):
    """Full lrcvt() (seeding -> 20 classify+update iterations -> final
    classify) on the GPU equals the reference's trajectory bit for bit."""
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, classify_isobands,
                                       label_components, lrcvt, synth_field)

    m = load_json(f"lloyd_{case}.json")
    arr = load_npz(f"lloyd_{case}.npz")
    grid = synth_field(m["kind"], tuple(m["dims"]), 0)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", m["iso"])))
    assert sha(labels.component) == m["labels"]["component"]
    tess, trace = lrcvt(grid, labels, SeedingParams(**m["params"]),
                        LloydParams(max_updates=m["iters"], ds_tolerance=1e-9))
    assert trace == m["trace"]
    assert np.array_equal(tess.site_positions(), arr["sites_hist"][-1])
    assert sha(tess.site_of) == m["final"]["site_of"]
    assert sha(tess.dist) == m["final"]["dist"]
    assert sha(tess.src) == m["final"]["src"]
    assert sha(tess.state) == m["final"]["state"]
    for k in ("rounds", "sweeps", "assigned"):
        assert tess.report[k] == m["final"]["report"][k]


@pytest.mark.slow
def test_c3_horseshoe256_trajectory_matches_reference():
    """BASELINE config C3 (256^3 horseshoe, 4097 sites, 20 updates): every
    iteration's sites and the final arrays equal the reference run."""
    _run_case("c3_horseshoe256")


def _run_case(case):
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, classify_isobands,
                                       label_components, lrcvt, synth_field)

    m = load_json(f"lloyd_{case}.json")
    arr = load_npz(f"lloyd_{case}.npz")
    grid = synth_field(m["kind"], tuple(m["dims"]), 0)
    assert sha(grid.fields["f"]) == m["f_sha"]
    labels = label_components(classify_isobands(grid, IsobandSpec("f", m["iso"])))
    assert sha(labels.component) == m["labels"]["component"]
    tess, trace = lrcvt(grid, labels, SeedingParams(**m["params"]),
                        LloydParams(max_updates=m["iters"], ds_tolerance=1e-9))
    assert trace == m["trace"]
    assert np.array_equal(tess.site_positions(), arr["sites_hist"][-1])
    assert sha(tess.site_of) == m["final"]["site_of"]
    assert sha(tess.dist) == m["final"]["dist"]
    assert sha(tess.src) == m["final"]["src"]


def test_audit_clean_on_seeded_volume():
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, audit_tessellation,
                                       classify_isobands, label_components, lrcvt, synth_field)

    grid = synth_field("spiral", (64, 64, 1), 0)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.3, 0.55, 0.8])))
    tess, _ = lrcvt(grid, labels, SeedingParams(alpha=200, seed=0), LloydParams(max_updates=10, ds_tolerance=1e-9))
    aud = audit_tessellation(tess, labels)
    for k in ("restriction_violations", "broken_chains", "chain_site_mismatch", "euclid_bound_violations",
              "nonfinite_dist", "segment_violations"):
        assert aud[k] == 0, (k, aud)
    assert aud["chain_depth_ok"]

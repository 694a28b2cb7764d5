"""CPU: pin the oracle (and the host-side seeding / synth restatements) to
golden vectors produced by the reference package itself
(tests/golden/make_golden.py). Bit-exact unless stated."""

import hashlib

import numpy as np
import pytest

from conftest import case_arrays, load_json, load_npz


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_classify_cases_bit_exact(classify_golden, oracle_mod):
    npz, meta = classify_golden
    for name, m in meta.items():
        a = case_arrays(npz, name)
        r = oracle_mod.classify(m["dims"], m["spacing"], a["comp"], a["site_pos"], a["site_comp"],
                                m["n_components"])
        assert r["bad"] == 0, name
        for key in ("site_of", "dist", "src", "state"):
            assert np.array_equal(r[key], a[key]), (name, key)
        assert r["rounds"] == m["report"]["rounds"], name
        assert r["sweeps"] == m["report"]["sweeps"], name
        assert r["assigned"] == m["report"]["assigned"], name


def test_centroidal_cases_bit_exact(classify_golden, oracle_mod):
    npz, meta = classify_golden
    for name, m in meta.items():
        a = case_arrays(npz, name)
        u = oracle_mod.centroidal(m["dims"], m["spacing"], a["comp"], a["site_of"], a["src"],
                                  a.get("weights"), a["site_pos"], a["site_comp"])
        assert np.array_equal(u["sums"], a["sums4"]), name
        assert np.array_equal(u["new_pos"], a["new_pos"]), name
        assert u["mean_ds"] == m["mean_ds"], name
        assert u["empty"] == m["empty_regions"], name
        phi, depth = oracle_mod.phi_chains(a["site_of"], a["src"])
        assert depth == m["max_chain_depth"], name


def test_site_outside_component_counted(oracle_mod):
    comp = np.zeros(64, np.int32)
    r = oracle_mod.classify((8, 8, 1), (1, 1, 1), comp, [[4.5, 4.5, 0.5]], [3], 4)
    assert r["bad"] == 1


def test_raycast_t_bit_exact(oracle_mod):
    npz, meta = load_npz("raycast.npz"), load_json("raycast.json")
    for name, m in meta.items():
        a = case_arrays(npz, name)
        got = [oracle_mod.segment_hit_t(a["comp"], m["dims"], m["spacing"], s[:3], s[3:], w)
               for s, w in zip(a["segs"], a["want"])]
        assert np.array_equal(np.array(got), a["t"]), name


def test_masks_restatement(oracle_mod):
    npz, meta = load_npz("masks.npz"), load_json("masks.json.gz")
    for name, m in meta.items():
        a = case_arrays(npz, name)
        if "f" not in a:
            continue
        layer = oracle_mod.isobands(a["f"], m["iso"])
        assert np.array_equal(layer, a["layer"]), name
        comp, table = oracle_mod.label_components(layer, m["dims"], len(m["iso"]) - 1)
        assert np.array_equal(comp, a["component"]), name
        assert [(t["id"], t["layer"], t["voxel_count"], t["bbox"]) for t in table] == \
               [(t["id"], t["layer"], t["voxel_count"], t["bbox"]) for t in m["table"]], name


def test_synth_fields_match_reference():
    from paper_2208_06970_b200.grid import synth_field

    meta = load_json("masks.json.gz")
    for name, kind, dims in (("rings40", "rings", (40, 40, 1)), ("spiral64", "spiral", (64, 64, 1)),
                             ("spiral48_3d", "spiral", (48, 40, 36)),
                             ("horseshoe64", "horseshoe", (64, 64, 1)),
                             ("smooth24", "random-smooth", (24, 24, 1))):
        seed = 1 if name == "rings40" else (3 if name == "smooth24" else 0)
        g = synth_field(kind, dims, seed)
        assert sha(g.fields["f"]) == meta[name]["f_sha"], name


def test_seeding_matches_reference(oracle_mod):
    from paper_2208_06970_b200.grid import LabelMap, synth_field
    from paper_2208_06970_b200.seeding import SeedingParams, seed_sites

    gold = load_json("seeding.json")
    for name, m in gold.items():
        g = synth_field(m["kind"], tuple(m["dims"]), 0)
        assert sha(g.fields["f"]) == m["f_sha"], name
        assert sha(g.fields["g"]) == m["g_sha"], name
        layer = oracle_mod.isobands(g.fields["f"], m["iso"])
        comp, table = oracle_mod.label_components(layer, m["dims"], len(m["iso"]) - 1)
        from paper_2208_06970_b200.grid import ComponentInfo

        labels = LabelMap(tuple(m["dims"]), layer, comp,
                          [ComponentInfo(t["id"], t["layer"], t["voxel_count"], tuple(t["bbox"]), (0, 0))
                           for t in table], m["iso"], "f")
        sites, rep = seed_sites(g, labels, SeedingParams(**m["params"]))
        assert [[*s.position, s.component_id] for s in sites] == m["sites"], name
        assert rep["target_counts"] == m["report"]["target_counts"], name


@pytest.mark.parametrize("case", ["spiral48_det", "smooth32_3d_g2", "c1_spiral256"])
def test_lloyd_trajectory_bit_exact(case, oracle_mod):
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap, synth_field
    from paper_2208_06970_b200.seeding import SeedingParams, seed_sites, voxel_weights

    m = load_json(f"lloyd_{case}.json")
    arr = load_npz(f"lloyd_{case}.npz")
    g = synth_field(m["kind"], tuple(m["dims"]), 0)
    layer = oracle_mod.isobands(g.fields["f"], m["iso"])
    comp, table = oracle_mod.label_components(layer, m["dims"], len(m["iso"]) - 1)
    assert sha(comp) == m["labels"]["component"]
    labels = LabelMap(tuple(m["dims"]), layer, comp,
                      [ComponentInfo(t["id"], t["layer"], t["voxel_count"], tuple(t["bbox"]), (0, 0))
                       for t in table], m["iso"], "f")
    params = SeedingParams(**m["params"])
    sites, _ = seed_sites(g, labels, params)
    pos0 = np.array([s.position for s in sites])
    hist_ref = arr["sites_hist"]
    assert np.array_equal(pos0, hist_ref[0])
    sc = np.array([s.component_id for s in sites], np.int32)
    w = voxel_weights(g, params) if params.weight_field else None
    final, trace, hist = oracle_mod.lloyd(m["dims"], (1.0, 1.0, 1.0), comp, len(table), pos0, sc, w,
                                          m["iters"], 1e-9)
    assert trace == m["trace"]
    assert len(hist) == len(hist_ref)
    for k, h in enumerate(hist):
        assert np.array_equal(h, hist_ref[k]), k
    assert np.array_equal(final["site_of"], arr["site_of"])
    assert np.array_equal(final["dist"], arr["dist"])
    assert np.array_equal(final["src"], arr["src"])


def test_aggregate_restatement_matches_reference(oracle_mod):
    gold = load_json("aggregate.json.gz")
    npz = load_npz("aggregate.npz")
    from paper_2208_06970_b200.grid import synth_field

    for name in ("explore", "stray"):
        m = gold[name]
        a = case_arrays(npz, name)
        if name == "explore":
            g = synth_field("spiral", (48, 48, 1), 0)
            fields = g.fields
        else:
            fields = {"f": a["f"], "g": a["g"]}
        layers = [t["layer"] for t in m["table"]]
        names = list(fields)
        pairs = [(x, y) for i, x in enumerate(names) for y in names[i:]]
        blobs = oracle_mod.aggregate_moments(fields, a["component"], a["site_of"], m["site_comp"], layers,
                                             m["n_layers"], pairs)
        assert len(blobs) == len(m["blobs"])
        for (scope, sid, agg), ref in zip(blobs, m["blobs"]):
            assert (scope, sid) == (ref["scope"], ref["id"])
            assert agg["n"] == ref["m"]["n"]
            assert agg["sums"] == ref["m"]["sums"]
            assert agg["min"] == ref["m"]["min"] and agg["max"] == ref["m"]["max"]


def test_histogram_restatement(oracle_mod):
    gold = load_json("aggregate.json.gz")["hist"]
    vals = load_npz("aggregate.npz")["hist/values"]
    for key, h in gold.items():
        counts, under, over = oracle_mod.histogram1d(vals, 64, h["lo"], h["hi"])
        assert counts.tolist() == h["counts"] and under == h["under"] and over == h["over"], key

"""GPU parity at the north-star volumes (SURVEY.md §8(c) strategy (4)).

C4 (512^3 random-smooth, 32 776 g-weighted sites): against digests written by
the REFERENCE itself in this container (tests/golden/make_golden.py --only
c4): the synthetic fields, masks and component table, the seeded sites, both
Lloyd iterations' sites / per-voxel arrays / report counters, the final
classification, and the per-cell aggregation (moments of the three field
pairs, 64-bin histograms). Tolerance: none for arrays, counts, ids, min/max
and histogram counts; power sums within 1e-12 relative (numpy's x**3 / x**4
may differ by an ulp from a correctly rounded product).

C5 (1024^3, 262 144 sites; the reference needs ~130 GB and cannot run in the
build container): one classification + centroidal update against the CPU
oracle port (oracle/lrcvt_oracle.c, itself pinned to the reference's golden
vectors) on the box, bit-exact, and the z-slab global mode with 2 emulated
slabs bit-identical to the single-domain run.
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import GOLDEN, load_json, load_npz

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _close(a, b, rtol=1e-12):
    return a == b or abs(a - b) <= rtol * max(abs(a), abs(b))


@pytest.fixture(scope="module")
def c4():
    from paper_2208_06970_b200 import (IsobandSpec, SeedingParams, classify_isobands, label_components, seed_sites,
                                       synth_field, voxel_weights)

    if not (GOLDEN / "lloyd_c4_smooth512.json").exists():
        pytest.skip("C4 golden not generated")
    m = load_json("lloyd_c4_smooth512.json")
    arr = load_npz("lloyd_c4_smooth512.npz")
    grid = synth_field(m["kind"], tuple(m["dims"]), 0)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", m["iso"])))
    params = SeedingParams(**m["params"])
    sites, _ = seed_sites(grid, labels, params, device=True)
    weights = voxel_weights(grid, params)
    return m, arr, grid, labels, params, sites, weights


def test_c4_inputs_masks_and_seeds_match_reference(c4):
    m, arr, grid, labels, params, sites, _ = c4
    assert sha(grid.fields["f"]) == m["f_sha"] and sha(grid.fields["g"]) == m["g_sha"]
    assert sha(labels.layer) == m["labels"]["layer"]
    assert sha(labels.component) == m["labels"]["component"]
    assert labels.n_components == m["labels"]["n_components"]
    for got, want in zip(labels.component_table, m["labels"]["table"]):
        assert got.id == want["id"] and got.layer == want["layer"] and got.voxel_count == want["voxel_count"]
        assert list(got.bbox) == list(want["bbox"])
    pos = np.array([s.position for s in sites])
    assert np.array_equal(pos, arr["sites_hist"][0])
    assert [s.component_id for s in sites] == m["site_comp"]


def test_c4_lloyd_iterations_match_reference(c4):
    """Two Lloyd iterations + the final classification through the public
    API (voronoi_classify -> read the four arrays -> centroidal_update):
    every iteration's arrays, counters and new sites equal the reference's."""
    from paper_2208_06970_b200 import centroidal_update, voronoi_classify

    m, arr, grid, labels, params, sites, weights = c4
    cur = sites
    for it in range(m["iters"]):
        tess = voronoi_classify(grid, labels, cur, weights)
        st = m["iter_stats"][it]
        for key in ("site_of", "dist", "src", "state"):
            assert sha(getattr(tess, key)) == st[key], (it, key)
        for key in ("rounds", "sweeps", "assigned"):
            assert tess.report[key] == st[key], (it, key)
        cur, mean_ds = centroidal_update(tess)
        assert mean_ds == m["trace"][it], it
        assert np.array_equal(np.array([s.position for s in cur]), arr["sites_hist"][it + 1]), it
        del tess
    final = voronoi_classify(grid, labels, cur, weights)
    for key in ("site_of", "dist", "src", "state"):
        assert sha(getattr(final, key)) == m["final"][key], key
    for key in ("rounds", "sweeps", "assigned"):
        assert final.report[key] == m["final"]["report"][key], key
    c4[0]["_final_tess"] = final  # reused by the aggregation test (same module)


def test_c4_aggregation_matches_reference(c4):
    import gzip
    import json

    from paper_2208_06970_b200 import aggregate_moments, centroidal_update, voronoi_classify
    from paper_2208_06970_b200.pipeline import aggregate_histograms

    m, arr, grid, labels, params, sites, weights = c4
    tess = m.get("_final_tess")
    if tess is None:  # run alone: rebuild the final state from the reference's final sites
        from paper_2208_06970_b200.seeding import Site

        cur = [Site(tuple(p), int(c)) for p, c in zip(arr["sites_hist"][-1], m["site_comp"])]
        tess = voronoi_classify(grid, labels, cur, weights)
        assert sha(tess.site_of) == m["final"]["site_of"]
    with gzip.open(GOLDEN / "aggregate_c4.json.gz", "rt") as fh:
        g = json.load(fh)
    blobs = aggregate_moments(grid, labels, tess)
    S = g["n_sites"]
    per_pair = len(blobs) // 3
    for k, (xn, yn) in enumerate(g["pairs"]):
        want = g[f"{xn}{yn}"]
        mine = blobs[k * per_pair:(k + 1) * per_pair]
        regions = [json.loads(b.payload) for b in mine[:S]]
        assert sha(np.array([r["n"] for r in regions], np.int64)) == want["n_sha"]
        mm = np.array([[r["min"][0], r["max"][0], r["min"][1], r["max"][1]] for r in regions], np.float64)
        assert sha(mm) == want["minmax_sha"]

        def same(a, b):
            assert a["n"] == b["n"] and a["min"] == b["min"] and a["max"] == b["max"]
            for key, v in b["sums"].items():
                assert _close(a["sums"][key], v), key

        for rid, blob in want["regions"].items():
            same(regions[int(rid)], blob)
        comps = [json.loads(b.payload) for b in mine[S:S + labels.n_components]]
        for cid, blob in want["components"].items():
            same(comps[int(cid)], blob)
        layers = [json.loads(b.payload) for b in mine[S + labels.n_components:]]
        assert len(layers) == len(want["layers"])
        for a, b in zip(layers, want["layers"]):
            same(a, b)
    h = aggregate_histograms(grid, labels, tess, fields=["f", "g"], bins=64)
    for nm in ("f", "g"):
        want = g["hist"][nm]
        assert h["axes"][nm] == (want["lo"], want["hi"])
        rows = np.array([np.concatenate([r.counts, [r.underflow, r.overflow]]) for r in h["region"][nm]],
                        np.int64)
        assert sha(rows) == want["sha"]


def test_c5_classify_update_vs_oracle_and_slabs():
    """1024^3 (C5 input of bench.py, 262 144 sites): one classification +
    centroidal update bit-exact against the CPU oracle port, and the 2-slab
    global mode (emulated on this GPU) bit-identical to the single domain."""
    import torch

    import bench
    from oracle import oracle
    from paper_2208_06970_b200.multigpu import Emulated, GlobalClassifier
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    cfg = bench.CONFIGS["c5"]
    grid, labels, params, sites, _ = bench.build_workload(cfg, 0)
    S = len(sites)
    assert S >= 262_000
    eng = engine_for(labels, grid.spacing, S)
    pos = np.array([s.position for s in sites])
    sc = np.array([s.component_id for s in sites], np.int32)
    pos_d = torch.from_numpy(pos).cuda()
    sc_d = torch.from_numpy(sc).cuda()
    st = eng.classify(pos_d, sc_d, want_state=True)
    mode, w_d = lloyd_weight_mode(torch, grid, params, None)
    vlen = voxel_length(grid.dims, grid.spacing)
    new_pos, disp, _, _ = eng.centroidal(pos_d, sc_d, mode, w_d, 0.5 * vlen)
    site_of, dist, src, state = eng.host_arrays()
    # the single-domain engine is released before the slab ranks take its memory (1024^3: ~30 GB per rank)
    del eng
    labels._b200_engine = None
    torch.cuda.empty_cache()
    # 2 emulated z-slabs over the same inputs
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, S, Emulated(2))
    gst = gc.classify(pos_d, sc_d)
    for r in gc.engines:
        v0, v1, e = gc.own_slab(r)
        ss_r = e.ss[v0:v1].cpu().numpy()
        assert np.array_equal(ss_r[:, 0], site_of[v0:v1]), r
        assert np.array_equal(ss_r[:, 1], src[v0:v1]), r
        assert np.array_equal(e.dist[v0:v1].cpu().numpy(), dist[v0:v1]), r
        assert np.array_equal(e.state[v0:v1].cpu().numpy(), state[v0:v1]), r
    g_pos, _, _ = gc.centroidal(pos_d, sc_d, mode, w_d, 0.5 * vlen)
    assert torch.equal(g_pos, new_pos)
    assert (gst["rounds"], gst["sweeps"], gst["evaluations"], gst["commits"]) == \
        (st["rounds"], st["sweeps"], st["evaluations"], st["commits"])
    del gc
    torch.cuda.empty_cache()
    # CPU oracle on the host copy of the same inputs
    oracle.build()
    import os

    oracle.set_num_threads(os.cpu_count() or 1)
    w = grid.fields["g"].astype(np.float64)  # voxel_weights with gamma 1
    ref = oracle.classify(grid.dims, grid.spacing, labels.component, pos, sc, labels.n_components)
    assert np.array_equal(site_of, ref["site_of"])
    assert np.array_equal(src, ref["src"])
    assert np.array_equal(dist, ref["dist"])
    assert np.array_equal(state, ref["state"])
    assert st["rounds"] == ref["rounds"] and st["sweeps"] == ref["sweeps"]
    assert st["evaluations"] == ref["evaluations"] and st["commits"] == ref["commits"]
    u = oracle.centroidal(grid.dims, grid.spacing, labels.component, ref["site_of"], ref["src"], w, pos, sc)
    assert np.array_equal(new_pos.cpu().numpy(), u["new_pos"])
    assert math.isclose(float(disp.cpu().numpy().mean() / vlen), u["mean_ds"], rel_tol=0, abs_tol=0)

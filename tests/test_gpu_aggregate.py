"""GPU parity: per-cell moment aggregation and histograms.

Tolerances: n, min, max, blob order and histogram counts bit-exact; power
sums within rtol 1e-12 of the reference's math.fsum (the GPU forms x^3, x^4
with correctly rounded products and sums them in compensated fp64; numpy's
x**3 / x**4 may differ from a correctly rounded product by an ulp, SURVEY.md
Appendix A.10)."""

import json

import numpy as np
import pytest

from conftest import case_arrays, load_json, load_npz

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def _labels(dims, comp, table, n_layers):
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap

    comp = np.ascontiguousarray(comp, dtype=np.int32)
    layer = np.full(comp.size, -1, np.int32)
    lay = {t["id"]: t["layer"] for t in table}
    for c, l in lay.items():
        layer[comp == c] = l
    infos = [ComponentInfo(t["id"], t["layer"], t["voxel_count"], tuple(t["bbox"]), tuple(t.get("band", (0, 0))))
             for t in table]
    return LabelMap(tuple(dims), layer, comp, infos, [float(i) for i in range(n_layers + 1)], "f")


def _tess(dims, site_of, site_comp, comp):
    from paper_2208_06970_b200 import Site, Tessellation

    n = site_of.size
    sites = [Site((0.5, 0.5, 0.5), int(c)) for c in site_comp]
    return Tessellation(tuple(dims), (1.0, 1.0, 1.0), np.ascontiguousarray(site_of, np.int32), np.zeros(n),
                        np.full(n, -1, np.int32), np.zeros(n, np.uint8), comp, sites, {})


def _check_blobs(got, ref):
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        m = json.loads(g.payload)
        rm = r["m"] if "m" in r else r[2]
        scope, sid = (r["scope"], r["id"]) if "scope" in r else (r[0], r[1])
        assert (g.scope, g.scope_id) == (scope, sid)
        assert m["n"] == rm["n"]
        assert m["min"] == rm["min"] and m["max"] == rm["max"]
        for k, v in rm["sums"].items():
            assert m["sums"][k] == pytest.approx(v, rel=RTOL, abs=1e-300), (scope, sid, k)


def test_aggregate_moments_golden():
    from paper_2208_06970_b200 import VoxelGrid, aggregate_moments, synth_field

    gold = load_json("aggregate.json.gz")
    npz = load_npz("aggregate.npz")
    for name in ("explore", "stray"):
        m = gold[name]
        a = case_arrays(npz, name)
        grid = synth_field("spiral", (48, 48, 1), 0) if name == "explore" else \
            VoxelGrid(tuple(m["dims"]), (1, 1, 1), {"f": a["f"], "g": a["g"]})
        labels = _labels(m["dims"], a["component"], m["table"], m["n_layers"])
        tess = _tess(m["dims"], a["site_of"], m["site_comp"], labels.component)
        _check_blobs(aggregate_moments(grid, labels, tess), m["blobs"])


@pytest.mark.parametrize("seed", [0, 1])
def test_aggregate_moments_vs_oracle(seed, oracle_mod):
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, aggregate_moments,
                                       classify_isobands, default_pairs, label_components, lrcvt, synth_field)

    grid = synth_field("random-smooth", (40, 36, 30), seed)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.3, 0.5, 0.7])))
    tess, _ = lrcvt(grid, labels, SeedingParams(alpha=60, seed=seed), LloydParams(max_updates=2))
    pairs = default_pairs(grid.field_names())
    got = aggregate_moments(grid, labels, tess, pairs)
    ref = oracle_mod.aggregate_moments(grid.fields, labels.component, tess.site_of,
                                       list(tess.site_components()), [c.layer for c in labels.component_table],
                                       labels.n_layers, pairs)
    _check_blobs(got, ref)


def test_aggregate_histograms_exact(oracle_mod):
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, VoxelGrid, aggregate_histograms,
                                       classify_isobands, label_components, lrcvt, synth_field)

    base = synth_field("gaussian-mix", (32, 30, 28), 2)
    # plant values exactly on the global bin edges to exercise the edge rule
    g = base.fields["g"].copy()
    f = base.fields["f"]
    lo, hi = float(g[f > 0.3].min()), float(g[f > 0.3].max())
    edges = np.linspace(lo, hi, 65).astype(np.float32)
    idx = np.flatnonzero(f > 0.3)[:: max(1, (f > 0.3).sum() // 400)][:len(edges) * 3]
    g[idx] = np.resize(edges, idx.size)
    grid = VoxelGrid(base.dims, base.spacing, {"f": f, "g": g})
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.3, 0.8])))
    tess, _ = lrcvt(grid, labels, SeedingParams(alpha=30, seed=1), LloydParams(max_updates=1))
    h = aggregate_histograms(grid, labels, tess, ["f", "g"], bins=64)
    inb = labels.component >= 0
    for nm in ("f", "g"):
        vals = grid.fields[nm].astype(np.float64)
        alo, ahi = h["axes"][nm]
        assert (alo, ahi) == (float(vals[inb].min()), float(vals[inb].max()))
        for r, hist in enumerate(h["region"][nm]):
            sel = vals[tess.site_of == r]
            counts, under, over = oracle_mod.histogram1d(sel, 64, alo, ahi)
            assert hist.counts.tolist() == counts.tolist(), (nm, r)
            assert (hist.underflow, hist.overflow) == (under, over)
        total = sum(hh.counts.sum() for hh in h["region"][nm]) + sum(hh.counts.sum() for hh in h["stray"][nm].values())
        assert total == inb.sum()


def test_histogram_fixed_axes_golden():
    """stats.histogram1d golden vectors (incl. values on edges) through the
    GPU binning rule: one cell holding all values."""
    from paper_2208_06970_b200 import Site, Tessellation, VoxelGrid, aggregate_histograms
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap

    gold = load_json("aggregate.json.gz")["hist"]
    vals = load_npz("aggregate.npz")["hist/values"].astype(np.float32)
    n = vals.size
    grid = VoxelGrid((n, 1, 1), (1, 1, 1), {"v": vals})
    comp = np.zeros(n, np.int32)
    labels = LabelMap((n, 1, 1), np.zeros(n, np.int32), comp, [ComponentInfo(0, 0, n, (0, 0, 0, n - 1, 0, 0), (0, 1))],
                      [0.0, 1.0], "v")
    tess = Tessellation((n, 1, 1), (1, 1, 1), np.zeros(n, np.int32), np.zeros(n), np.arange(n, dtype=np.int32),
                        np.zeros(n, np.uint8), comp, [Site((0.5, 0.5, 0.5), 0)], {})
    for key, h in gold.items():
        out = aggregate_histograms(grid, labels, tess, ["v"], bins=64, axes={"v": (h["lo"], h["hi"])})
        hist = out["region"]["v"][0]
        assert hist.counts.tolist() == h["counts"], key
        assert (hist.underflow, hist.overflow) == (h["under"], h["over"]), key

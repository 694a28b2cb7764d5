"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package itself (lrcvt 0.1.0, /root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_ref \
        python tests/golden/make_golden.py [--big]

The outputs are committed; the reference itself never travels to the GPU box
and nothing at test/bench time imports it. Small cases store full arrays;
large cases (C2 128^3, C3 256^3) store sha256 digests of the reference arrays,
the per-iteration site positions and the mean_ds trace, which the tests
recompute from regenerated inputs.
"""

from __future__ import annotations

import argparse
import gzip
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref():
    import lrcvt  # noqa: F401  (fails loudly when PYTHONPATH is not set)
    from lrcvt import _kernels as K
    from lrcvt import grid as G
    from lrcvt import pipeline as P
    from lrcvt import seeding as S
    from lrcvt import stats as ST
    from lrcvt import tessellation as T

    return G, S, T, P, ST, K


def rect(G, nx, ny, nz=1, spacing=(1.0, 1.0, 1.0)):
    f = np.full(nx * ny * nz, 0.5, np.float32)
    grid = G.VoxelGrid((nx, ny, nz), spacing, {"f": f})
    labels = G.label_components(G.classify_isobands(grid, G.IsobandSpec("f", [0.0, 1.0])))
    return grid, labels


def classify_cases(G, S, T):
    """(name, grid, labels, sites, weights) tuples covering the reference's
    own classify/centroid tests (test_tessellation.py) plus seeded 2D/3D
    volumes."""
    out = []
    g, l = rect(G, 21, 13)
    out.append(("rect21x13", g, l, [S.Site((10.5, 6.5, 0.5), 0)], None))
    g, l = rect(G, 40, 30)
    rng = np.random.default_rng(17)
    vox = rng.choice(g.size, 10, replace=False)
    out.append(("rect40x30", g, l, [S.Site((v % 40 + 0.5, v // 40 + 0.5, 0.5), 0) for v in vox], None))
    g, l = rect(G, 50, 40)
    rng = np.random.default_rng(123)
    pts = rng.uniform((0.5, 0.5), (49.5, 39.5), size=(25, 2))
    out.append(("convex50x40", g, l, [S.Site((float(x), float(y), 0.5), 0) for x, y in pts], None))
    g, l = rect(G, 9, 1)
    out.append(("tie9x1", g, l, [S.Site((2.5, 0.5, 0.5), 0), S.Site((6.5, 0.5, 0.5), 0)], None))
    g, l = rect(G, 11, 11)
    out.append(("square11", g, l, [S.Site((2.5, 8.5, 0.5), 0)], None))
    out.append(("square11_fixed", g, l, [S.Site((5.5, 5.5, 0.5), 0)], None))
    g, l = rect(G, 11, 1)
    w = np.ones(11)
    w[8:] = 50.0
    out.append(("weighted11", g, l, [S.Site((5.5, 0.5, 0.5), 0)], w))
    f = np.full(20 * 7, 0.5, np.float32)
    g = G.VoxelGrid((20, 7, 1), (0.5, 2.0, 1.0), {"f": f})
    l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", [0.0, 1.0])))
    out.append(("aniso20x7", g, l, [S.Site((5.25, 7.0, 0.5), 0)], None))
    n = 12
    f = np.full(n * n, 0.5, np.float32)
    f.reshape(1, n, n)[0][0 : n // 2, n // 2 :] = 0.0
    g = G.VoxelGrid((n, n, 1), (1, 1, 1), {"f": f})
    l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", [0.0, 1.0])))
    out.append(("lshape12", g, l, [S.Site((2.5, 2.5, 0.5), 0)], None))
    f = np.zeros(100, np.float32)
    f.reshape(1, 10, 10)[0, 0:2, :] = 0.5
    f.reshape(1, 10, 10)[0, 5:7, :] = 0.5
    g = G.VoxelGrid((10, 10, 1), (1, 1, 1), {"f": f})
    l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", [0.4, 0.6])))
    out.append(("twocomp10", g, l, [S.Site((0.5, 0.5, 0.5), 0)], None))
    g = G.synth_field("horseshoe", (64, 64, 1), 0)
    l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", [0.0, 0.12])))
    out.append(("u64", g, l, [S.Site((32 - 14.08, 9.0, 0.5), 0), S.Site((32 + 14.08, 9.0, 0.5), 0)], None))
    seeded = [
        ("spiral64", "spiral", (64, 64, 1), [0.3, 0.55, 0.8], dict(alpha=60, seed=5, weight_field="g")),
        ("horseshoe128", "horseshoe", (128, 128, 1), [0.0, 0.12, 0.3], dict(alpha=40, seed=4)),
        ("smooth24_3d", "random-smooth", (24, 24, 24), [0.35, 0.75], dict(alpha=30, seed=7)),
        ("spiral32_3d", "spiral", (32, 32, 32), [0.55, 0.75, 0.95], dict(alpha=60, seed=1, weight_field="g", gamma=2.0)),
        ("horseshoe40_3d", "horseshoe", (40, 40, 40), [0.0, 0.12, 0.3], dict(alpha=50, seed=2)),
        ("gmix32_3d", "gaussian-mix", (32, 32, 32), [0.3, 0.7], dict(alpha=40, seed=0, weight_field="g")),
    ]
    for name, kind, dims, iso, sp in seeded:
        g = G.synth_field(kind, dims, 0)
        l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", iso)))
        params = S.SeedingParams(**sp)
        sites, _ = S.seed_sites(g, l, params)
        out.append((name, g, l, sites, S.voxel_weights(g, params)))
    return out


def dump_classify(G, S, T, K):
    from lrcvt.tessellation import audit_tessellation

    arrays = {}
    meta = {}
    for name, g, l, sites, w in classify_cases(G, S, T):
        tess = T.voronoi_classify(g, l, sites, w)
        new_sites, mean_ds = T.centroidal_update(tess)
        aud = audit_tessellation(tess, l)
        sp = np.array([s.position for s in sites], np.float64).reshape(-1, 3)
        sc = np.array([s.component_id for s in sites], np.int32)
        arrays[f"{name}/comp"] = l.component
        arrays[f"{name}/site_pos"] = sp
        arrays[f"{name}/site_comp"] = sc
        if w is not None:
            arrays[f"{name}/weights"] = np.asarray(w, np.float64)
        arrays[f"{name}/site_of"] = tess.site_of
        arrays[f"{name}/dist"] = tess.dist
        arrays[f"{name}/src"] = tess.src
        arrays[f"{name}/state"] = tess.state
        arrays[f"{name}/new_pos"] = np.array([s.position for s in new_sites], np.float64).reshape(-1, 3)
        phi, depth = K._phi_chains(tess.site_of, tess.src)
        wv = np.ones(g.size) if w is None else np.asarray(w, np.float64)
        wsum, tx, ty, tz = K._centroid_targets(
            l.component, g.dims[0], g.dims[1], *g.spacing, tess.site_of, phi, wv, len(sites))
        arrays[f"{name}/sums4"] = np.stack([wsum, tx, ty, tz])
        meta[name] = {
            "dims": list(g.dims),
            "spacing": list(g.spacing),
            "n_components": l.n_components,
            "report": {k: tess.report[k] for k in ("rounds", "sweeps", "assigned", "components_without_sites")},
            "mean_ds": mean_ds,
            "empty_regions": tess.report["empty_regions"],
            "max_chain_depth": int(depth),
            "audit": {k: (int(v) if not isinstance(v, bool) else v) for k, v in aud.items()},
        }
    np.savez_compressed(OUT / "classify.npz", **arrays)
    (OUT / "classify.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


def dump_raycast(G, K):
    arrays, meta = {}, {}
    for name, dims, seed, iso, spacing in (
        ("smooth48", (48, 48, 1), 11, [0.35, 0.75], (1.0, 1.0, 1.0)),
        ("smooth20_3d", (20, 20, 20), 11, [0.35, 0.75], (1.0, 1.0, 1.0)),
        ("smooth16_aniso", (16, 12, 10), 3, [0.3, 0.7], (0.5, 1.25, 2.0)),
    ):
        g = G.synth_field("random-smooth", dims, seed)
        l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", iso)))
        rng = np.random.default_rng(5)
        nx, ny, nz = dims
        ext = np.array(dims) * np.array(spacing)
        segs = []
        for _ in range(400):
            a = rng.uniform(0.0, 1.0, 3) * ext
            if rng.random() < 0.5:  # voxel-centre starts, like the kernels use
                a = (np.floor(a / spacing) + 0.5) * spacing
            b = rng.uniform(-0.2, 1.2, 3) * ext if rng.random() < 0.2 else rng.uniform(0.0, 1.0, 3) * ext
            if nz == 1:
                a[2] = b[2] = 0.5 * spacing[2]
            segs.append(np.concatenate([a, b]))
        segs = np.array(segs)
        ts = []
        wants = []
        for s in segs:
            cx = min(max(int(np.floor(s[0] / spacing[0])), 0), nx - 1)
            cy = min(max(int(np.floor(s[1] / spacing[1])), 0), ny - 1)
            cz = min(max(int(np.floor(s[2] / spacing[2])), 0), nz - 1)
            want = int(l.component[cx + nx * (cy + ny * cz)])
            wants.append(want)
            ts.append(K._segment_hit_t(l.component, nx, ny, nz, *spacing, *s, want))
        arrays[f"{name}/comp"] = l.component
        arrays[f"{name}/segs"] = segs
        arrays[f"{name}/want"] = np.array(wants, np.int32)
        arrays[f"{name}/t"] = np.array(ts, np.float64)
        meta[name] = {"dims": list(dims), "spacing": list(spacing)}
    np.savez_compressed(OUT / "raycast.npz", **arrays)
    (OUT / "raycast.json").write_text(json.dumps(meta, indent=1))


def table_json(l):
    return [
        {"id": c.id, "layer": c.layer, "voxel_count": c.voxel_count, "bbox": list(c.bbox), "band": list(c.band)}
        for c in l.component_table
    ]


def dump_masks(G):
    arrays, meta = {}, {}
    cases = []
    for seed in (0, 1, 2):
        rng = np.random.default_rng(seed)
        dims = (32, 32, 32)
        f = rng.random(np.prod(dims)).astype(np.float32)
        cases.append((f"random32_s{seed}", G.VoxelGrid(dims, (1, 1, 1), {"f": f}), [0.3, 0.6, 0.9], True))
    cases.append(("rings40", G.synth_field("rings", (40, 40, 1), 1), [0.2, 0.5, 0.8], False))
    cases.append(("spiral64", G.synth_field("spiral", (64, 64, 1), 0), [0.3, 0.55, 0.8], False))
    cases.append(("spiral48_3d", G.synth_field("spiral", (48, 40, 36), 0), [0.55, 0.75, 0.95], False))
    cases.append(("horseshoe64", G.synth_field("horseshoe", (64, 64, 1), 0), [0.0, 0.12], False))
    cases.append(("smooth24", G.synth_field("random-smooth", (24, 24, 1), 3), [0.3, 0.7], False))
    cases.append(("halfopen", G.VoxelGrid((4, 1, 1), (1, 1, 1), {"f": np.array([0.25, 0.75, 0.1, 0.9], np.float32)}), [0.25, 0.75], True))
    cases.append(("diag2x2", G.VoxelGrid((2, 2, 1), (1, 1, 1), {"f": np.array([0.5, 0, 0, 0.5], np.float32)}), [0.4, 0.6], True))
    cases.append(("empty4", G.VoxelGrid((2, 2, 1), (1, 1, 1), {"f": np.full(4, 0.5, np.float32)}), [0.6, 0.7], True))
    for name, g, iso, store_field in cases:
        lm = G.classify_isobands(g, G.IsobandSpec("f", iso))
        l = G.label_components(lm)
        if store_field:
            arrays[f"{name}/f"] = g.fields["f"]
        arrays[f"{name}/layer"] = l.layer
        arrays[f"{name}/component"] = l.component
        meta[name] = {"dims": list(g.dims), "iso": iso, "table": table_json(l), "f_sha": sha(g.fields["f"])}
    np.savez_compressed(OUT / "masks.npz", **arrays)
    with gzip.open(OUT / "masks.json.gz", "wt") as fh:
        json.dump(meta, fh)


def blobs_json(blobs):
    return [{"scope": b.scope, "id": b.scope_id, "kind": b.kind, "m": json.loads(b.payload)} for b in blobs]


def dump_aggregate(G, S, T, P, ST):
    out = {}
    grid = G.synth_field("spiral", (48, 48, 1), 0)
    iso = G.IsobandSpec("f", [0.3, 0.55, 0.8])
    res = P.run_pipeline(grid, iso, S.SeedingParams(alpha=40, seed=7), T.LloydParams(max_updates=6, ds_tolerance=0.05))
    arrays = {"explore/site_of": res.tess.site_of, "explore/component": res.labels.component}
    out["explore"] = {
        "dims": list(grid.dims),
        "site_comp": [int(s.component_id) for s in res.tess.sites],
        "table": table_json(res.labels),
        "n_layers": res.labels.n_layers,
        "blobs": blobs_json(P.aggregate_moments(grid, res.labels, res.tess)),
    }
    # stray voxels: a component whose only site is removed -> unassigned voxels
    nx, ny = 30, 12
    f = np.zeros(nx * ny, dtype=np.float32)
    f3 = f.reshape(1, ny, nx)[0]
    f3[2:5, 2:12] = 0.3
    f3[2:5, 18:28] = 0.3
    f3[7:10, 6:24] = 0.7
    gg = np.linspace(0, 1, nx * ny, dtype=np.float32)
    grid2 = G.VoxelGrid((nx, ny, 1), (1.0, 1.0, 1.0), {"f": f, "g": gg})
    labels2 = G.label_components(G.classify_isobands(grid2, G.IsobandSpec("f", [0.1, 0.5, 0.9])))
    sites = [S.Site((3.5, 3.5, 0.5), 0), S.Site((8.5, 3.5, 0.5), 0), S.Site((10.5, 8.5, 0.5), 2)]
    tess2 = T.voronoi_classify(grid2, labels2, sites)
    arrays["stray/f"] = f
    arrays["stray/g"] = gg
    arrays["stray/site_of"] = tess2.site_of
    arrays["stray/component"] = labels2.component
    out["stray"] = {
        "dims": [nx, ny, 1],
        "site_comp": [0, 0, 2],
        "table": table_json(labels2),
        "n_layers": labels2.n_layers,
        "blobs": blobs_json(P.aggregate_moments(grid2, labels2, tess2)),
    }
    # histograms (stats.py:194-203), including values exactly on edges
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.random(5000), np.linspace(0.1, 0.9, 65), [0.1, 0.9, 0.0, 1.0]])
    vals32 = vals.astype(np.float32).astype(np.float64)
    hist = {}
    for key, v, lo, hi in (("unit", vals32, 0.1, 0.9), ("auto", vals32, None, None), ("tight", vals32, 0.25, 0.2500001)):
        h = ST.histogram1d(v, bins=64, lo=lo, hi=hi)
        hist[key] = {"lo": h.lo, "hi": h.hi, "counts": h.counts.tolist(), "under": h.underflow, "over": h.overflow}
    arrays["hist/values"] = vals32
    out["hist"] = hist
    np.savez_compressed(OUT / "aggregate.npz", **arrays)
    with gzip.open(OUT / "aggregate.json.gz", "wt") as fh:
        json.dump(out, fh)


def dump_seeding(G, S):
    out = {}
    for name, kind, dims, iso, sp in (
        ("spiral64", "spiral", (64, 64, 1), [0.3, 0.55, 0.8], dict(alpha=60, seed=5, weight_field="g")),
        ("spiral256_c1", "spiral", (256, 256, 1), [0.3, 0.55, 0.8], dict(alpha=64, gamma=1.0, weight_field="g", block_size=16, seed=0)),
        ("smooth24_3d", "random-smooth", (24, 24, 24), [0.35, 0.75], dict(alpha=30, seed=7)),
        ("gmix32_g2", "gaussian-mix", (32, 32, 32), [0.3, 0.7], dict(alpha=40, seed=0, weight_field="g", gamma=2.0, block_size=8)),
        ("rings40_many", "rings", (40, 40, 1), [0.2, 0.5, 0.8], dict(alpha=900, seed=3, block_size=4)),
    ):
        g = G.synth_field(kind, dims, 0)
        l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", iso)))
        sites, rep = S.seed_sites(g, l, S.SeedingParams(**sp))
        out[name] = {
            "kind": kind, "dims": list(dims), "iso": iso, "params": sp,
            "f_sha": sha(g.fields["f"]), "g_sha": sha(g.fields["g"]),
            "sites": [[*s.position, s.component_id] for s in sites],
            "report": {k: (v if not isinstance(v, dict) else {str(a): b for a, b in v.items()}) for k, v in rep.items()},
        }
    (OUT / "seeding.json").write_text(json.dumps(out))


def lloyd_trajectory(G, S, T, grid, labels, params, lloyd, full_arrays):
    """Restates lrcvt() (tessellation.py:251-275) step by step so every
    iteration's sites and arrays can be recorded."""
    sites, _ = S.seed_sites(grid, labels, params)
    weights = S.voxel_weights(grid, params)
    rec = {"sites": [[list(s.position) for s in sites]], "trace": [], "iter_stats": []}
    for _ in range(lloyd.max_updates):
        t0 = time.time()
        tess = T.voronoi_classify(grid, labels, sites, weights)
        t1 = time.time()
        sites, mean_ds = T.centroidal_update(tess)
        t2 = time.time()
        rec["trace"].append(mean_ds)
        rec["sites"].append([list(s.position) for s in sites])
        rec["iter_stats"].append({
            "site_of": sha(tess.site_of), "dist": sha(tess.dist), "src": sha(tess.src),
            "rounds": tess.report["rounds"], "sweeps": tess.report["sweeps"],
            "classify_s": t1 - t0, "update_s": t2 - t1,
        })
        if mean_ds < lloyd.ds_tolerance:
            break
    final = T.voronoi_classify(grid, labels, sites, weights)
    rec["final"] = {"site_of": sha(final.site_of), "dist": sha(final.dist), "src": sha(final.src),
                    "state": sha(final.state), "report": {k: final.report[k] for k in ("rounds", "sweeps", "assigned")}}
    rec["site_comp"] = [s.component_id for s in sites]
    rec["labels"] = {"layer": sha(labels.layer), "component": sha(labels.component), "n_components": labels.n_components}
    rec["f_sha"] = sha(grid.fields["f"])
    rec["g_sha"] = sha(grid.fields["g"])
    arrays = {"sites_hist": np.array(rec.pop("sites"), dtype=np.float64)}
    if full_arrays:
        arrays.update(site_of=final.site_of, dist=final.dist, src=final.src)
    return rec, arrays


def dump_lloyd(G, S, T, big: bool):
    cases = [
        ("c1_spiral256", "spiral", (256, 256, 1), [0.3, 0.55, 0.8],
         dict(alpha=64, gamma=1.0, weight_field="g", block_size=16, seed=0), 20, True),
        ("spiral48_det", "spiral", (48, 48, 1), [0.3, 0.7], dict(alpha=60, seed=3), 3, True),
        ("smooth32_3d_g2", "random-smooth", (32, 32, 32), [0.35, 0.75],
         dict(alpha=80, seed=1, weight_field="g", gamma=2.0), 6, True),
    ]
    if big:
        cases += [
            ("c2_gmix128", "gaussian-mix", (128, 128, 128), [0.3, 0.7],
             dict(alpha=512, weight_field="g", seed=0), 20, False),
            ("c3_horseshoe256", "horseshoe", (256, 256, 256), [0.0, 0.12, 0.3],
             dict(alpha=4096, seed=0), 20, False),
        ]
    for name, kind, dims, iso, sp, iters, full in cases:
        t0 = time.time()
        g = G.synth_field(kind, dims, 0)
        l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", iso)))
        rec, arrays = lloyd_trajectory(G, S, T, g, l, S.SeedingParams(**sp),
                                       T.LloydParams(max_updates=iters, ds_tolerance=1e-9), full)
        rec.update(kind=kind, dims=list(dims), iso=iso, params=sp, iters=iters)
        (OUT / f"lloyd_{name}.json").write_text(json.dumps(rec))
        np.savez_compressed(OUT / f"lloyd_{name}.npz", **arrays)
        print(f"{name}: {time.time() - t0:.1f}s", file=sys.stderr)


def c4_aggregates(G, ST, grid, labels, tess, every=64, bins=64):
    """C4 per-cell aggregation (pipeline.py:187-238) with the reference's own
    stats.accumulate / merge / histogram1d. The region selection
    `in_band[region == rid]` is taken from one stable argsort by site instead of
    S boolean scans (the selected index arrays are identical, so every
    accumulate call sees the same samples in the same order); at 512^3 the
    O(S * N_in) scan of aggregate_moments itself would take days.
    Stored: sha256 of the exact per-region n / min / max arrays, full blobs of
    every `every`-th region, all component and layer blobs, and 64-bin
    histograms of f and g per cell on the global in-band [min, max] axes
    (sha of the full count table + the sampled rows)."""
    in_band = np.nonzero(labels.component != -1)[0]
    comp = labels.component[in_band]
    region = tess.site_of[in_band]
    order = np.argsort(region, kind="stable")
    sreg = region[order]
    nS = len(tess.sites)
    starts = np.searchsorted(sreg, np.arange(nS), side="left")
    ends = np.searchsorted(sreg, np.arange(nS), side="right")
    unassigned = in_band[region == -1]
    site_comp = tess.site_components()
    layer_of_comp = {c.id: c.layer for c in labels.component_table}
    pairs = [("f", "f"), ("f", "g"), ("g", "g")]
    out = {"every": every, "pairs": pairs, "n_sites": nS}
    for xn, yn in pairs:
        fx = grid.fields[xn].astype(np.float64)
        fy = grid.fields[yn].astype(np.float64)
        region_aggs = []
        for rid in range(nS):
            sel = in_band[order[starts[rid]:ends[rid]]]
            region_aggs.append(ST.accumulate(np.stack([fx[sel], fy[sel]], axis=1), xn, yn))
        stray = {}
        if unassigned.size:
            uc = labels.component[unassigned]
            for c in np.unique(uc):
                sel = unassigned[uc == c]
                stray[int(c)] = ST.accumulate(np.stack([fx[sel], fy[sel]], axis=1), xn, yn)
        comp_aggs = {}
        for info in labels.component_table:
            agg = ST.MomentAggregate(x_name=xn, y_name=yn)
            for rid in np.nonzero(site_comp == info.id)[0]:
                agg = ST.merge(agg, region_aggs[int(rid)])
            if info.id in stray:
                agg = ST.merge(agg, stray[info.id])
            comp_aggs[info.id] = agg
        layer_aggs = []
        for li in range(labels.n_layers):
            agg = ST.MomentAggregate(x_name=xn, y_name=yn)
            for cid, a in comp_aggs.items():
                if layer_of_comp[cid] == li:
                    agg = ST.merge(agg, a)
            layer_aggs.append(agg)
        key = f"{xn}{yn}"
        out[key] = {
            "n_sha": sha(np.array([a.n for a in region_aggs], np.int64)),
            "minmax_sha": sha(np.array([[a.min_x, a.max_x, a.min_y, a.max_y] for a in region_aggs], np.float64)),
            "regions": {str(r): region_aggs[r].to_dict() for r in range(0, nS, every)},
            "stray": {str(c): a.to_dict() for c, a in stray.items()},
            "components": {str(c): a.to_dict() for c, a in comp_aggs.items()},
            "layers": [a.to_dict() for a in layer_aggs],
        }
        print(f"  c4 aggregate {key} done", file=sys.stderr, flush=True)
    hist = {}
    for nm in ("f", "g"):
        v = grid.fields[nm].astype(np.float64)
        lo, hi = float(v[in_band].min()), float(v[in_band].max())
        rows = np.zeros((nS, bins + 2), np.int64)
        for rid in range(nS):
            sel = in_band[order[starts[rid]:ends[rid]]]
            h = ST.histogram1d(v[sel], bins=bins, lo=lo, hi=hi)
            rows[rid, :bins] = h.counts
            rows[rid, bins] = h.underflow
            rows[rid, bins + 1] = h.overflow
        hist[nm] = {"lo": lo, "hi": hi, "sha": sha(rows),
                    "rows": {str(r): rows[r].tolist() for r in range(0, nS, every)}}
    out["hist"] = hist
    return out


def dump_c4(G, S, T, ST):
    """C4: 512^3 random-smooth, iso [0.35, 0.5, 0.65, 0.8],
    alpha 32768, weight 'g'; two Lloyd iterations + the final classify
    recorded as digests, then the per-cell aggregation of the final state.
    ~17 GB RSS, tens of minutes in this container."""
    t0 = time.time()
    kind, dims, iso = "random-smooth", (512, 512, 512), [0.35, 0.5, 0.65, 0.8]
    sp = dict(alpha=32768, weight_field="g", seed=0)
    g = G.synth_field(kind, dims, 0)
    print(f"c4 synth {time.time() - t0:.0f}s", file=sys.stderr, flush=True)
    l = G.label_components(G.classify_isobands(g, G.IsobandSpec("f", iso)))
    print(f"c4 labels {time.time() - t0:.0f}s", file=sys.stderr, flush=True)
    params = S.SeedingParams(**sp)
    sites, _ = S.seed_sites(g, l, params)
    weights = S.voxel_weights(g, params)
    rec = {"sites": [[list(s.position) for s in sites]], "trace": [], "iter_stats": []}
    for it in range(2):
        t1 = time.time()
        tess = T.voronoi_classify(g, l, sites, weights)
        t2 = time.time()
        sites, mean_ds = T.centroidal_update(tess)
        rec["trace"].append(mean_ds)
        rec["sites"].append([list(s.position) for s in sites])
        rec["iter_stats"].append({"site_of": sha(tess.site_of), "dist": sha(tess.dist), "src": sha(tess.src),
                                  "state": sha(tess.state), "rounds": tess.report["rounds"],
                                  "sweeps": tess.report["sweeps"], "assigned": tess.report["assigned"],
                                  "classify_s": t2 - t1, "update_s": time.time() - t2})
        print(f"c4 iteration {it}: classify {t2 - t1:.0f}s", file=sys.stderr, flush=True)
        del tess
    final = T.voronoi_classify(g, l, sites, weights)
    rec["final"] = {"site_of": sha(final.site_of), "dist": sha(final.dist), "src": sha(final.src),
                    "state": sha(final.state),
                    "report": {k: final.report[k] for k in ("rounds", "sweeps", "assigned")}}
    rec["site_comp"] = [s.component_id for s in sites]
    rec["labels"] = {"layer": sha(l.layer), "component": sha(l.component), "n_components": l.n_components,
                     "table": table_json(l)}
    rec["f_sha"] = sha(g.fields["f"])
    rec["g_sha"] = sha(g.fields["g"])
    rec.update(kind=kind, dims=list(dims), iso=iso, params=sp, iters=2)
    arrays = {"sites_hist": np.array(rec.pop("sites"), dtype=np.float64)}
    np.savez_compressed(OUT / "lloyd_c4_smooth512.npz", **arrays)
    (OUT / "lloyd_c4_smooth512.json").write_text(json.dumps(rec))
    print(f"c4 lloyd done {time.time() - t0:.0f}s", file=sys.stderr, flush=True)
    agg = c4_aggregates(G, ST, g, l, final)
    with gzip.open(OUT / "aggregate_c4.json.gz", "wt") as fh:
        json.dump(agg, fh)
    print(f"c4 all done {time.time() - t0:.0f}s", file=sys.stderr, flush=True)


def dump_blocks(G, S, T, P):
    """Block-mode run_pipeline (pipeline.py:45-160) results for the
    distributed block driver."""
    arrays, meta = {}, {}
    for name, kind, dims, iso, sp, lp, blocks in (
        ("spiral48_b221", "spiral", (48, 48, 1), [0.3, 0.55, 0.8], dict(alpha=40, seed=7),
         dict(max_updates=6, ds_tolerance=0.05), (2, 2, 1)),
        ("smooth24_b112", "random-smooth", (24, 24, 24), [0.35, 0.75], dict(alpha=30, seed=3, weight_field="g"),
         dict(max_updates=3, ds_tolerance=1e-9), (1, 1, 2)),
        ("gmix20_b212", "gaussian-mix", (20, 18, 16), [0.3, 0.7], dict(alpha=25, seed=1),
         dict(max_updates=2, ds_tolerance=1e-9), (2, 1, 2)),
    ):
        g = G.synth_field(kind, dims, 0)
        res = P.run_pipeline(g, G.IsobandSpec("f", iso), S.SeedingParams(**sp), T.LloydParams(**lp), blocks)
        for key in ("site_of", "dist", "src", "state"):
            arrays[f"{name}/{key}"] = getattr(res.tess, key)
        arrays[f"{name}/layer"] = res.labels.layer
        arrays[f"{name}/component"] = res.labels.component
        arrays[f"{name}/sites"] = np.array([[*s.position, s.component_id] for s in res.tess.sites])
        meta[name] = {"kind": kind, "dims": list(dims), "iso": iso, "seeding": sp, "lloyd": lp,
                      "blocks": list(blocks), "trace": res.trace, "block_traces": res.block_traces,
                      "table": table_json(res.labels)}
    np.savez_compressed(OUT / "blocks.npz", **arrays)
    (OUT / "blocks.json").write_text(json.dumps(meta))


def dump_layout(G, S, T, P):
    """.lrcvt files written by the reference's build_and_write (layout.py:123-219):
    sha256 of the file, of its record block and of the manifest, the summary,
    plus the inputs (arrays in layout.npz) so the tests can rebuild them."""
    import tempfile

    from lrcvt import layout as LY

    cases = {}
    grid = G.synth_field("spiral", (48, 48, 1), 0)
    res = P.run_pipeline(grid, G.IsobandSpec("f", [0.3, 0.55, 0.8]), S.SeedingParams(alpha=40, seed=7),
                         T.LloydParams(max_updates=4, ds_tolerance=0.05))
    cases["explore"] = (grid, res.labels, res.tess, P.aggregate_moments(grid, res.labels, res.tess))
    # unassigned voxels inside the record order (a component without sites)
    nx, ny = 30, 12
    f = np.zeros(nx * ny, dtype=np.float32)
    f3 = f.reshape(ny, nx)
    f3[2:5, 2:12] = 0.3
    f3[2:5, 18:28] = 0.3
    f3[7:10, 6:24] = 0.7
    g2 = G.VoxelGrid((nx, ny, 1), (1.0, 1.0, 1.0), {"f": f, "g": np.linspace(0, 1, nx * ny, dtype=np.float32)})
    l2 = G.label_components(G.classify_isobands(g2, G.IsobandSpec("f", [0.1, 0.5, 0.9])))
    t2 = T.voronoi_classify(g2, l2, [S.Site((3.5, 3.5, 0.5), 0), S.Site((8.5, 3.5, 0.5), 0),
                                     S.Site((10.5, 8.5, 0.5), 2)])
    cases["stray"] = (g2, l2, t2, P.aggregate_moments(g2, l2, t2))
    # 3D, anisotropic spacing, two bands, every site of component 1 dropped
    g3 = G.VoxelGrid((24, 20, 16), (1.0, 0.5, 2.0), G.synth_field("random-smooth", (24, 20, 16), 0).fields)
    l3 = G.label_components(G.classify_isobands(g3, G.IsobandSpec("f", [0.35, 0.5, 0.7])))
    sites3, _ = S.seed_sites(g3, l3, S.SeedingParams(alpha=30, seed=2))
    sites3 = [s for s in sites3 if s.component_id != 1]
    t3 = T.voronoi_classify(g3, l3, sites3)
    cases["smooth3d"] = (g3, l3, t3, [])
    arrays, out = {}, {}
    with tempfile.TemporaryDirectory() as d:
        for name, (grid, labels, tess, blobs) in cases.items():
            path = Path(d) / f"{name}.lrcvt"
            summary = LY.build_and_write(grid, labels, tess, blobs, path)
            data = path.read_bytes()
            man = Path(str(path) + ".manifest.json").read_text()
            h = LY.LayoutReader(path).header
            for k, v in grid.fields.items():
                arrays[f"{name}/field/{k}"] = v
            arrays[f"{name}/layer"] = labels.layer
            arrays[f"{name}/component"] = labels.component
            arrays[f"{name}/site_of"] = tess.site_of
            summary.pop("path")
            out[name] = {
                "dims": list(grid.dims), "spacing": list(grid.spacing), "fields": grid.field_names(),
                "iso_field": labels.field_name, "iso_values": list(labels.iso_values),
                "table": table_json(labels),
                "sites": [[*s.position, s.component_id] for s in tess.sites],
                "blobs": [{"scope": b.scope, "id": b.scope_id, "kind": b.kind, "payload": b.payload.decode()}
                          for b in blobs],
                "file_sha": hashlib.sha256(data).hexdigest(),
                "data_sha": hashlib.sha256(data[h.data_off:h.agg_off]).hexdigest(),
                "manifest_sha": hashlib.sha256(man.encode()).hexdigest(),
                "file_bytes": len(data), "summary": summary,
            }
    np.savez_compressed(OUT / "layout.npz", **arrays)
    (OUT / "layout.json").write_text(json.dumps(out))


def dump_sitegraph(G, S, T):
    """sitegraph.py region_adjacency / all_pairs_paths / fold_metric on the
    layout cases (inputs from layout.npz/json) and a 3D Lloyd result."""
    from lrcvt import sitegraph as SG

    meta = json.loads((OUT / "layout.json").read_text())
    arr = np.load(OUT / "layout.npz")
    tess = {}
    for name, m in meta.items():
        sites = [S.Site(tuple(s[:3]), int(s[3])) for s in m["sites"]]
        n = int(np.prod(m["dims"]))
        tess[name] = T.Tessellation(tuple(m["dims"]), tuple(m["spacing"]), arr[f"{name}/site_of"], np.zeros(n),
                                    np.zeros(n, np.int32), np.zeros(n, np.uint8), arr[f"{name}/component"], sites)
    grid = G.synth_field("gaussian-mix", (32, 30, 28), 0)
    labels = G.label_components(G.classify_isobands(grid, G.IsobandSpec("f", [0.25, 0.5, 0.75])))
    t, _ = T.lrcvt(grid, labels, S.SeedingParams(alpha=80, weight_field="g", seed=4), T.LloydParams(max_updates=3))
    tess["gmix3d"] = t
    out, arrays = {}, {}
    for name, tt in tess.items():
        gr = SG.region_adjacency(tt)
        paths = SG.all_pairs_paths(gr)
        fm = SG.fold_metric(gr.positions, paths, c=1.5)
        if name == "gmix3d":
            arrays["gmix3d/site_of"] = tt.site_of
            arrays["gmix3d/component"] = tt.component
            arrays["gmix3d/sites"] = np.array([[*s.position, s.component_id] for s in tt.sites])
        out[name] = {"edges": gr.edges.tolist(), "weights": [w.hex() for w in gr.weights],
                     "paths_sha": sha(paths), "fold_sha": sha(fm.matrix), "dims": list(tt.dims)}
    np.savez_compressed(OUT / "sitegraph.npz", **arrays)
    (OUT / "sitegraph.json").write_text(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also record C2 128^3 and C3 256^3 trajectories")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    G, S, T, P, ST, K = ref()
    todo = a.only.split(",") if a.only else ["classify", "raycast", "masks", "aggregate", "seeding", "lloyd",
                                             "blocks", "layout", "sitegraph"]
    if "classify" in todo:
        dump_classify(G, S, T, K)
    if "raycast" in todo:
        dump_raycast(G, K)
    if "masks" in todo:
        dump_masks(G)
    if "aggregate" in todo:
        dump_aggregate(G, S, T, P, ST)
    if "seeding" in todo:
        dump_seeding(G, S)
    if "lloyd" in todo:
        dump_lloyd(G, S, T, a.big)
    if "blocks" in todo:
        dump_blocks(G, S, T, P)
    if "layout" in todo:
        dump_layout(G, S, T, P)
    if "sitegraph" in todo:
        dump_sitegraph(G, S, T)
    if "c4" in todo:  # only on request (--only c4): tens of minutes, ~17 GB
        dump_c4(G, S, T, ST)


if __name__ == "__main__":
    main()

"""Site adjacency graph (sitegraph.py:46-128 of the reference; SURVEY.md §8(f)
rank 4) against the reference's own outputs (tests/golden/sitegraph.json):
edges bit-exact, weights bit-exact (same numpy expression), all-pairs paths
and the fold matrix by sha256. CPU: oracle + host graph functions; GPU: the
device face scan."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _cases():
    meta = json.loads((GOLD / "sitegraph.json").read_text())
    lay = json.loads((GOLD / "layout.json").read_text())
    la = np.load(GOLD / "layout.npz")
    sa = np.load(GOLD / "sitegraph.npz")
    from paper_2208_06970_b200.seeding import Site
    from paper_2208_06970_b200.tessellation import Tessellation

    out = {}
    for name, m in meta.items():
        if name in lay:
            site_of, comp = la[f"{name}/site_of"], la[f"{name}/component"]
            sites = [Site(tuple(s[:3]), int(s[3])) for s in lay[name]["sites"]]
            spacing = tuple(lay[name]["spacing"])
        else:
            site_of, comp = sa[f"{name}/site_of"], sa[f"{name}/component"]
            sites = [Site(tuple(s[:3]), int(s[3])) for s in sa[f"{name}/sites"]]
            spacing = (1.0, 1.0, 1.0)
        dims = tuple(m["dims"])
        n = int(np.prod(dims))
        z = np.zeros(n)
        out[name] = (m, Tessellation(dims, spacing, site_of, z, z.astype(np.int32), z.astype(np.uint8), comp, sites))
    return out


NAMES = ["explore", "stray", "smooth3d", "gmix3d"]


def _check_graph(m, tess, edges):
    from paper_2208_06970_b200.sitegraph import SiteGraph, all_pairs_paths, fold_metric

    assert edges.tolist() == m["edges"]
    pos = tess.site_positions()
    w = np.linalg.norm(pos[edges[:, 0]] - pos[edges[:, 1]], axis=1) if edges.size else np.empty(0)
    assert [x.hex() for x in w] == m["weights"]
    g = SiteGraph(tess.n_sites, edges, w, tess.site_components(), pos)
    paths = all_pairs_paths(g)
    assert _sha(paths) == m["paths_sha"]
    assert _sha(fold_metric(pos, paths, c=1.5).matrix) == m["fold_sha"]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_and_host_graph_match_reference(name, oracle_mod):
    m, tess = _cases()[name]
    edges = oracle_mod.region_adjacency_edges(tess.dims, tess.site_of, tess.component)
    _check_graph(m, tess, edges)


def test_fold_metric_rejects_small_c():
    from paper_2208_06970_b200.sitegraph import fold_metric

    with pytest.raises(ValueError):
        fold_metric(np.zeros((2, 3)), np.zeros((2, 2)), c=0.5)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_region_adjacency_matches_reference(name):
    from paper_2208_06970_b200.sitegraph import region_adjacency

    m, tess = _cases()[name]
    g = region_adjacency(tess)
    _check_graph(m, tess, g.edges)
    assert [x.hex() for x in g.weights] == m["weights"]


@pytest.mark.gpu
def test_gpu_region_adjacency_fresh_vs_oracle(oracle_mod):
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, classify_isobands,
                                       label_components, lrcvt, synth_field)
    from paper_2208_06970_b200.sitegraph import region_adjacency

    for kind, dims, iso, alpha in (("horseshoe", (48, 40, 36), [0.0, 0.12, 0.3], 150),
                                   ("spiral", (160, 120, 1), [0.3, 0.55, 0.8], 90)):
        grid = synth_field(kind, dims, 0)
        labels = label_components(classify_isobands(grid, IsobandSpec("f", iso)))
        tess, _ = lrcvt(grid, labels, SeedingParams(alpha=alpha, seed=2), LloydParams(max_updates=2))
        g = region_adjacency(tess)
        ref = oracle_mod.region_adjacency_edges(tess.dims, tess.site_of, tess.component)
        assert np.array_equal(g.edges, ref), kind

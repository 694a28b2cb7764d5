"""Site adjacency graph, all-pairs path distances and the fold metric
(reference ``lrcvt.sitegraph``, sitegraph.py:1-128).

The O(N) part -- scanning every voxel face for pairs of different sites in one
component -- runs on the GPU (``lrcvt_region_adjacency``: one streaming pass,
warp-deduplicated inserts into a device hash set, compaction + radix sort).
The graph itself is O(sites): edge weights (the reference's
``np.linalg.norm`` expression), Dijkstra per component (scipy) and the fold
ratio stay on the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np


@dataclass
class SiteGraph:
    n_sites: int
    edges: np.ndarray  # (E, 2) int64 site pairs, lo < hi, sorted
    weights: np.ndarray  # (E,) Euclidean site-to-site distances
    site_components: np.ndarray  # (n_sites,)
    positions: np.ndarray  # (n_sites, 3)

    def to_dict(self) -> dict:
        return {"n_sites": self.n_sites, "edges": self.edges.tolist(), "weights": self.weights.tolist()}


@dataclass
class FoldMetric:
    matrix: np.ndarray  # (n, n); 0 on the diagonal, c for disconnected pairs
    c: float
    site_components: np.ndarray = field(default=None)


def _site_of_device(torch, tess):
    dev = tess.device_state() if hasattr(tess, "device_state") else None
    if dev is not None:
        return dev[0][:, 0].contiguous()
    return torch.from_numpy(np.ascontiguousarray(tess.site_of, dtype=np.int32)).to("cuda")


def region_adjacency(tess) -> SiteGraph:
    """Sites whose regions share a voxel face inside one component
    (sitegraph.py:46-82); the face scan runs on the GPU."""
    from . import _lib

    torch = _lib.require_cuda()
    L = _lib.lib()
    nx, ny, nz = tess.dims
    site_of = _site_of_device(torch, tess)
    comp = torch.from_numpy(np.ascontiguousarray(tess.component, dtype=np.int32)).to("cuda")
    n = tess.n_sites
    cap = max(16, 16 * n)
    for _ in range(3):
        edges_d = torch.empty((cap, 2), dtype=torch.int64, device="cuda")
        got = ctypes.c_int64()
        rc = L.lrcvt_region_adjacency(nx, ny, nz, site_of.data_ptr(), comp.data_ptr(), n, cap, edges_d.data_ptr(),
                                      ctypes.byref(got), _lib.stream_handle(torch))
        if rc == _lib.E_ARG and got.value > cap:
            cap = int(got.value)
            continue
        _lib.check(rc, "lrcvt_region_adjacency")
        break
    e = edges_d[: int(got.value)].cpu().numpy()
    pos = tess.site_positions()
    w = np.linalg.norm(pos[e[:, 0]] - pos[e[:, 1]], axis=1) if e.size else np.empty(0)
    return SiteGraph(n_sites=n, edges=e, weights=w, site_components=tess.site_components(), positions=pos)


def all_pairs_paths(graph: SiteGraph) -> np.ndarray:
    """Shortest-path distances over the site graph, inf across components;
    Dijkstra per component block (sitegraph.py:85-108)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra

    n = graph.n_sites
    out = np.full((n, n), np.inf)
    np.fill_diagonal(out, 0.0)
    if n == 0:
        return out
    adj = csr_matrix((graph.weights, (graph.edges[:, 0], graph.edges[:, 1])), shape=(n, n))
    for c in np.unique(graph.site_components):
        idx = np.nonzero(graph.site_components == c)[0]
        if idx.size > 1:
            out[np.ix_(idx, idx)] = dijkstra(adj[idx][:, idx], directed=False)
    return out


def fold_metric(positions: np.ndarray, path_dists: np.ndarray, c: float = 1.0) -> FoldMetric:
    """Straight-line over path distance per site pair, c where no path
    exists, 0 on the diagonal (sitegraph.py:111-128)."""
    if c < 1.0:
        raise ValueError("c must be >= 1")
    p = np.asarray(positions, dtype=np.float64)
    straight = np.linalg.norm(p[:, None, :] - p[None, :, :], axis=2)
    with np.errstate(invalid="ignore", divide="ignore"):
        ratio = np.where(np.isfinite(path_dists) & (path_dists > 0), straight / path_dists, c)
    np.fill_diagonal(ratio, 0.0)
    return FoldMetric(matrix=ratio, c=c)

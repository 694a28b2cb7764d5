"""End-to-end drivers: block-decomposed tessellation and per-cell aggregation.

Mirrors the reference's ``lrcvt.pipeline`` (pipeline.py:31-238):
``run_pipeline`` (block mode: axis-aligned blocks tessellated independently,
block faces act as restrictions), ``default_pairs`` and ``aggregate_moments``.
The per-cell power sums run on the GPU (csrc/aggregate.cuh); the roll-up of
region aggregates into components and layers is the reference's sequential
``merge`` on the host (tiny: S x 15 numbers), so blobs follow the reference's
order and merge arithmetic exactly.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import NONE_ID, ComponentInfo, IsobandSpec, LabelMap, VoxelGrid, classify_isobands, label_components
from .layout import AggregateBlob
from .seeding import SeedingParams, Site
from .stats import ORDERS, Histogram1D, MomentAggregate, merge
from .tessellation import LloydParams, Tessellation, lrcvt


@dataclass
class PipelineResult:
    grid: VoxelGrid
    labels: LabelMap
    tess: Tessellation
    trace: list[float]
    block_traces: list[list[float]] = field(default_factory=list)


def block_ranges(n: int, parts: int) -> list[tuple[int, int]]:
    """pipeline.py:40-42: np.linspace split, empty ranges dropped."""
    edges = np.linspace(0, n, parts + 1).astype(int)
    return [(int(edges[i]), int(edges[i + 1])) for i in range(parts) if edges[i] < edges[i + 1]]


def block_list(dims, blocks) -> list[tuple[tuple[int, int], tuple[int, int], tuple[int, int]]]:
    """Blocks in the reference's z -> y -> x processing order (pipeline.py:79-81)."""
    nx, ny, nz = dims
    rx, ry, rz = block_ranges(nx, blocks[0]), block_ranges(ny, blocks[1]), block_ranges(nz, blocks[2])
    return [(bx, by, bz) for bz in rz for by in ry for bx in rx]


def _combine_traces(block_traces: list[list[float]]) -> list[float]:
    if not block_traces:
        return []
    out = []
    for i in range(max(len(t) for t in block_traces)):
        out.append(float(np.mean([t[i] for t in block_traces if i < len(t)])))
    return out


def tessellate_block(grid: VoxelGrid, iso: IsobandSpec, seeding: SeedingParams, lloyd: LloydParams,
                     block, total_in_band: int, comp_off: int, label_fn=None, lloyd_fn=None):
    """One block of pipeline.py:82-108: sub-grid, local labels, alpha share,
    GPU Lloyd loop. Returns (sub_labels, tess, trace) or None when the block
    has no component."""
    sub = sub_grid(grid, block)
    sub_labels = (label_fn or gpu_label)(sub, iso)
    if sub_labels.n_components == 0:
        return None
    sub_seed = block_seeding(seeding, sub_labels.in_band_count(), total_in_band, comp_off)
    tess, trace = (lloyd_fn or lrcvt)(sub, sub_labels, sub_seed, lloyd)
    return sub, sub_labels, tess, trace


def run_pipeline(grid: VoxelGrid, iso: IsobandSpec, seeding: SeedingParams, lloyd: LloydParams,
                 blocks: tuple[int, int, int] = (1, 1, 1), label_fn=None, lloyd_fn=None) -> PipelineResult:
    """pipeline.py:45-160. blocks == (1,1,1): one tessellation of the whole
    grid. Otherwise each block is an independent LSRCVT (block faces are
    restrictions) merged with component/site id offsets in block order."""
    label_fn = label_fn or gpu_label
    lloyd_fn = lloyd_fn or lrcvt
    if tuple(blocks) == (1, 1, 1):
        labels = label_fn(grid, iso)
        tess, trace = lloyd_fn(grid, labels, seeding, lloyd)
        return PipelineResult(grid, labels, tess, trace, [trace])
    total_in_band = 0
    for block in block_list(grid.dims, blocks):
        total_in_band += label_fn(sub_grid(grid, block), iso).in_band_count()
    n = grid.size
    nx, ny, _ = grid.dims
    out = {
        "layer": np.full(n, NONE_ID, dtype=np.int32), "component": np.full(n, NONE_ID, dtype=np.int32),
        "site_of": np.full(n, NONE_ID, dtype=np.int32), "dist": np.full(n, np.inf),
        "src": np.full(n, NONE_ID, dtype=np.int32), "state": np.zeros(n, dtype=np.uint8),
    }
    table: list[ComponentInfo] = []
    sites: list[Site] = []
    block_traces: list[list[float]] = []
    comp_off = site_off = 0
    for block in block_list(grid.dims, blocks):
        res = tessellate_block(grid, iso, seeding, lloyd, block, total_in_band, comp_off, label_fn, lloyd_fn)
        if res is None:
            continue
        sub, sub_labels, tess, trace = res
        block_traces.append(trace)
        comp_off, site_off = merge_block(grid, block, sub_labels, tess, out, table, sites, comp_off, site_off)
    labels = LabelMap(dims=grid.dims, layer=out["layer"], component=out["component"], component_table=table,
                      iso_values=list(iso.iso_values), field_name=iso.field_name)
    merged = Tessellation(dims=grid.dims, spacing=grid.spacing, site_of=out["site_of"], dist=out["dist"],
                          src=out["src"], state=out["state"], component=out["component"], sites=sites,
                          report={"blocks": tuple(blocks), "n_blocks": len(block_traces)})
    return PipelineResult(grid, labels, merged, _combine_traces(block_traces), block_traces)


def sub_grid(grid: VoxelGrid, block) -> VoxelGrid:
    (x0, x1), (y0, y1), (z0, z1) = block
    nx, ny, nz = grid.dims
    return VoxelGrid((x1 - x0, y1 - y0, z1 - z0), grid.spacing,
                     {name: np.ascontiguousarray(arr.reshape(nz, ny, nx)[z0:z1, y0:y1, x0:x1]).ravel()
                      for name, arr in grid.fields.items()})


def gpu_label(sub: VoxelGrid, iso: IsobandSpec) -> LabelMap:
    return label_components(classify_isobands(sub, iso))


def block_seeding(seeding: SeedingParams, in_band: int, total_in_band: int, comp_off: int) -> SeedingParams:
    """pipeline.py:91-105: alpha is a global budget shared by in-band voxel
    count; per-block sampling streams offset by the running component count."""
    return SeedingParams(alpha=max(seeding.alpha * in_band / max(total_in_band, 1), 1e-9), gamma=seeding.gamma,
                         weight_field=seeding.weight_field, block_size=seeding.block_size,
                         seed=seeding.seed + comp_off)


def run_pipeline_distributed(grid: VoxelGrid, iso: IsobandSpec, seeding: SeedingParams, lloyd: LloydParams,
                             blocks: tuple[int, int, int], label_fn=gpu_label, lloyd_fn=lrcvt,
                             group=None, dst: int = 0) -> PipelineResult | None:
    """Block mode over torch.distributed ranks (one GPU each), the reference's
    own distributed semantics (pipeline.py:45-160): block b is
    tessellated by rank b % world with no data-path communication. Control
    exchanges only: one all_gather of per-block (component count, in-band
    count) fixes total_in_band and the component-id offsets that seed each
    block's RNG stream, and a final gather brings block results to `dst`,
    which merges them in the reference's block order. Returns the merged
    PipelineResult on `dst` (bit-identical to run_pipeline), None elsewhere.
    label_fn / lloyd_fn default to the GPU kernels."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    blist = block_list(grid.dims, blocks)
    mine = [b for b in range(len(blist)) if b % world == rank]
    local = {}
    for b in mine:
        sub = sub_grid(grid, blist[b])
        lab = label_fn(sub, iso)
        local[b] = (sub, lab)
    counts = {b: (local[b][1].n_components, local[b][1].in_band_count()) for b in mine}
    gathered: list = [None] * world
    dist.all_gather_object(gathered, counts, group=group)
    allc = {b: c for d in gathered for b, c in d.items()}
    total_in_band = sum(c[1] for c in allc.values())
    comp_off_of, off = {}, 0
    for b in range(len(blist)):
        comp_off_of[b] = off
        off += allc[b][0]
    results = {}
    for b in mine:
        sub, lab = local[b]
        if lab.n_components == 0:
            continue
        tess, trace = lloyd_fn(sub, lab, block_seeding(seeding, lab.in_band_count(), total_in_band,
                                                       comp_off_of[b]), lloyd)
        results[b] = (_portable_labels(lab), _portable_tess(tess), trace)
    out_list: list = [None] * world if rank == dst else None
    dist.gather_object(results, out_list, dst=dst, group=group)
    if rank != dst:
        return None
    allr = {b: r for d in out_list for b, r in d.items()}
    n = grid.size
    out = {
        "layer": np.full(n, NONE_ID, dtype=np.int32), "component": np.full(n, NONE_ID, dtype=np.int32),
        "site_of": np.full(n, NONE_ID, dtype=np.int32), "dist": np.full(n, np.inf),
        "src": np.full(n, NONE_ID, dtype=np.int32), "state": np.zeros(n, dtype=np.uint8),
    }
    table: list[ComponentInfo] = []
    sites: list[Site] = []
    block_traces: list[list[float]] = []
    comp_off = site_off = 0
    for b in range(len(blist)):
        if b not in allr:
            continue
        lab, tess, trace = allr[b]
        block_traces.append(trace)
        comp_off, site_off = merge_block(grid, blist[b], lab, tess, out, table, sites, comp_off, site_off)
    labels = LabelMap(dims=grid.dims, layer=out["layer"], component=out["component"], component_table=table,
                      iso_values=list(iso.iso_values), field_name=iso.field_name)
    merged = Tessellation(dims=grid.dims, spacing=grid.spacing, site_of=out["site_of"], dist=out["dist"],
                          src=out["src"], state=out["state"], component=out["component"], sites=sites,
                          report={"blocks": tuple(blocks), "n_blocks": len(block_traces)})
    return PipelineResult(grid, labels, merged, _combine_traces(block_traces), block_traces)


def _portable_labels(lab: LabelMap) -> LabelMap:
    """Plain LabelMap without cached device objects, for pickling."""
    return LabelMap(lab.dims, np.asarray(lab.layer), np.asarray(lab.component), list(lab.component_table),
                    list(lab.iso_values), lab.field_name)


def _portable_tess(t: Tessellation) -> Tessellation:
    """Plain-numpy copy (device-resident tessellations materialised) for pickling."""
    return Tessellation(t.dims, t.spacing, np.asarray(t.site_of), np.asarray(t.dist), np.asarray(t.src),
                        np.asarray(t.state), np.asarray(t.component), list(t.sites), dict(t.report), None)


def merge_block(grid, block, sub_labels, tess, out, table, sites, comp_off, site_off):
    """Scatter one block's result into the global arrays (pipeline.py:109-148)."""
    (x0, x1), (y0, y1), (z0, z1) = block
    nx, ny, _ = grid.dims
    sx, sy, sz = grid.spacing
    snx, sny = x1 - x0, y1 - y0
    lidx = np.arange(tess.site_of.size)
    gidx = (lidx % snx + x0) + nx * (((lidx // snx) % sny + y0) + ny * (lidx // (snx * sny) + z0))
    in_band = sub_labels.component != NONE_ID
    out["layer"][gidx[in_band]] = sub_labels.layer[in_band]
    out["component"][gidx[in_band]] = sub_labels.component[in_band] + comp_off
    assigned = tess.site_of != NONE_ID
    out["site_of"][gidx[assigned]] = tess.site_of[assigned] + site_off
    out["dist"][gidx[assigned]] = tess.dist[assigned]
    out["src"][gidx[assigned]] = gidx[tess.src[assigned]]
    out["state"][gidx] = tess.state
    for info in sub_labels.component_table:
        bb = info.bbox
        table.append(ComponentInfo(id=info.id + comp_off, layer=info.layer, voxel_count=info.voxel_count,
                                   bbox=(bb[0] + x0, bb[1] + y0, bb[2] + z0, bb[3] + x0, bb[4] + y0, bb[5] + z0),
                                   band=info.band))
    for s in tess.sites:
        sites.append(Site(position=(s.position[0] + x0 * sx, s.position[1] + y0 * sy, s.position[2] + z0 * sz),
                          component_id=s.component_id + comp_off))
    return comp_off + sub_labels.n_components, site_off + len(tess.sites)


# ---------------------------------------------------------------------------
# aggregation


def default_pairs(field_names: list[str]) -> list[tuple[str, str]]:
    """All unordered field pairs including self-pairs (pipeline.py:178-184)."""
    return [(a, b) for i, a in enumerate(field_names) for b in field_names[i:]]


def cell_aggregates_device(fields_d: list, comp_d, site_d, n_sites: int, n_comp: int,
                           pair_idx: np.ndarray, bins: int = 0, axes: np.ndarray | None = None) -> dict:
    """Device-resident per-cell pass (lrcvt_aggregate) on CUDA tensors:
    fields_d float32[N] each, comp_d / site_d int32[N]. Returns CUDA tensors
    count[C], sums[C, P, 15], minmax[C, P, 4] (+ hist[C, F, bins + 2]) and the
    axes actually used (numpy [F, 2])."""
    torch = _lib.require_cuda()
    L = _lib.lib()
    n_cells = n_sites + n_comp
    P, F = len(pair_idx), len(fields_d)
    C = max(n_cells, 1)
    count = torch.zeros(C, dtype=torch.int64, device="cuda")
    sums = torch.zeros((C, P, 15), dtype=torch.float64, device="cuda")
    minmax = torch.zeros((C, P, 4), dtype=torch.float64, device="cuda")
    hist = torch.zeros((C, F, bins + 2), dtype=torch.int64, device="cuda") if bins else None
    ptrs = (ctypes.c_void_p * F)(*[f.data_ptr() for f in fields_d])
    pr = np.ascontiguousarray(pair_idx, dtype=np.int32)
    ax = np.full((F, 2), np.nan) if axes is None else np.array(axes, dtype=np.float64).reshape(F, 2).copy()
    _lib.check(L.lrcvt_aggregate(int(comp_d.numel()), F, ptrs, comp_d.data_ptr(), site_d.data_ptr(), n_sites,
                                 n_comp, P, pr.ctypes.data, bins, ax.ctypes.data, count.data_ptr(),
                                 sums.data_ptr(), minmax.data_ptr(), hist.data_ptr() if hist is not None else None,
                                 _lib.stream_handle(torch)), "lrcvt_aggregate")
    return {"n_cells": n_cells, "count": count, "sums": sums, "minmax": minmax, "hist": hist, "axes": ax}


def cell_aggregates(grid: VoxelGrid, labels: LabelMap, site_of: np.ndarray, n_sites: int,
                    pairs: list[tuple[str, str]], bins: int = 0, axes=None) -> dict:
    """GPU per-cell pass from host arrays. Cells 0..S-1 are regions, S + c is
    the unassigned remainder of component c. Returns numpy arrays."""
    torch = _lib.require_cuda()
    names: list[str] = []
    for a, b in pairs:
        for nm in (a, b):
            if nm not in names:
                names.append(nm)
    for nm in names:
        if nm not in grid.fields:
            raise KeyError(f"unknown field '{nm}'; grid has {grid.field_names()}")
    fields_d = [torch.from_numpy(grid.fields[nm]).to("cuda") for nm in names]
    comp_d = torch.from_numpy(np.ascontiguousarray(labels.component, dtype=np.int32)).to("cuda")
    site_d = torch.from_numpy(np.ascontiguousarray(site_of, dtype=np.int32)).to("cuda")
    n_comp = labels.n_components
    if labels.component.size and labels.component.max() >= n_comp:
        n_comp = int(labels.component.max()) + 1
    pr = np.array([[names.index(a), names.index(b)] for a, b in pairs], dtype=np.int32)
    ax = np.full((len(names), 2), np.nan)
    if axes is not None:
        for i, nm in enumerate(names):
            if nm in axes:
                ax[i] = axes[nm]
    d = cell_aggregates_device(fields_d, comp_d, site_d, n_sites, n_comp, pr, bins, ax)
    n_cells = d["n_cells"]
    out = {"names": names, "n_cells": n_cells, "count": d["count"].cpu().numpy()[:n_cells],
           "sums": d["sums"].cpu().numpy()[:n_cells], "minmax": d["minmax"].cpu().numpy()[:n_cells],
           "axes": d["axes"]}
    if d["hist"] is not None:
        out["hist"] = d["hist"].cpu().numpy()[:n_cells]
    return out


def _agg_from(cells: dict, cell: int, k: int, x_name: str, y_name: str) -> MomentAggregate:
    agg = MomentAggregate(x_name=x_name, y_name=y_name, n=int(cells["count"][cell]))
    s = cells["sums"][cell, k]
    for t, (p, q) in enumerate(ORDERS):
        agg.sums[p, q] = s[t]
    mm = cells["minmax"][cell, k]
    agg.min_x, agg.max_x, agg.min_y, agg.max_y = (float(v) for v in mm)
    return agg


def aggregate_moments(grid: VoxelGrid, labels: LabelMap, tess: Tessellation,
                      pairs: list[tuple[str, str]] | None = None) -> list[AggregateBlob]:
    """Per-region moment aggregates rolled up to components and layers by
    merging, one set per variable pair (pipeline.py:187-238)."""
    pairs = pairs or default_pairs(grid.field_names())
    S = len(tess.sites)
    cells = cell_aggregates(grid, labels, tess.site_of, S, pairs)
    site_comp = tess.site_components()
    layer_of_comp = {c.id: c.layer for c in labels.component_table}
    by_comp: dict[int, list[int]] = {}
    for rid in range(S):
        by_comp.setdefault(int(site_comp[rid]), []).append(rid)
    blobs: list[AggregateBlob] = []
    for k, (x_name, y_name) in enumerate(pairs):
        region_aggs = [_agg_from(cells, rid, k, x_name, y_name) for rid in range(S)]
        blobs.extend(AggregateBlob.moments("region", rid, a) for rid, a in enumerate(region_aggs))
        comp_aggs: dict[int, MomentAggregate] = {}
        for info in labels.component_table:
            agg = MomentAggregate(x_name=x_name, y_name=y_name)
            for rid in by_comp.get(info.id, []):
                agg = merge(agg, region_aggs[rid])
            stray = S + info.id
            if stray < cells["n_cells"] and cells["count"][stray] > 0:
                agg = merge(agg, _agg_from(cells, stray, k, x_name, y_name))
            comp_aggs[info.id] = agg
            blobs.append(AggregateBlob.moments("component", info.id, agg))
        for li in range(labels.n_layers):
            agg = MomentAggregate(x_name=x_name, y_name=y_name)
            for cid, a in comp_aggs.items():
                if layer_of_comp[cid] == li:
                    agg = merge(agg, a)
            blobs.append(AggregateBlob.moments("layer", li, agg))
    return blobs


def aggregate_histograms(grid: VoxelGrid, labels: LabelMap, tess: Tessellation,
                         fields: list[str] | None = None, bins: int = 64,
                         axes: dict | None = None) -> dict:
    """Per-region histograms of each field on fixed global axes (default:
    in-band min / max, stats.py:186-191), binned with stats.histogram1d's
    numpy rule so they merge exactly across regions, blocks and GPUs.
    Returns {"axes": {field: (lo, hi)}, "region": {field: [Histogram1D]*S},
    "stray": {field: {component: Histogram1D}}}."""
    fields = fields or grid.field_names()
    S = len(tess.sites)
    cells = cell_aggregates(grid, labels, tess.site_of, S, [(f, f) for f in fields], bins=bins, axes=axes)
    out = {"axes": {}, "region": {}, "stray": {}}
    for i, nm in enumerate(cells["names"]):
        lo, hi = (float(v) for v in cells["axes"][i])
        out["axes"][nm] = (lo, hi)
        h = cells["hist"][:, i]
        out["region"][nm] = [Histogram1D(lo, hi, h[r, :bins].copy(), int(h[r, bins]), int(h[r, bins + 1]))
                             for r in range(S)]
        out["stray"][nm] = {c: Histogram1D(lo, hi, h[S + c, :bins].copy(), int(h[S + c, bins]),
                                           int(h[S + c, bins + 1]))
                            for c in range(cells["n_cells"] - S) if cells["count"][S + c] > 0}
    return out

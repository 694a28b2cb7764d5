"""The .lrcvt hierarchical layout (reference ``lrcvt.layout``, layout.py:1-488;
SURVEY.md §8(f) rank 2).

File = header, layer / component / region index tables, the record block
(in-band voxels ordered by layer, component, region, voxel; each record
{u32 x, y, z; f32 field[m]}, little-endian), then tagged aggregate blobs. A
JSON manifest mirrors the indexes.

B200 split: the O(N) part -- selecting the in-band voxels, ordering them by
(component, region, voxel) and packing the record block -- is one device pass
(``lrcvt_layout_records``: CUB select + a stable 64-bit radix sort + a
coalesced word-per-thread pack), which also yields every component's record
range and each record's region key. The host assembles the small index
tables and streams the bytes to disk. Region ranges use ``np.searchsorted``
over the region keys exactly as the reference does (layout.py:181-182; the
key sequence is only sorted per component, so the binary-search semantics
matter and are kept).
"""

from __future__ import annotations

import ctypes
import json
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .grid import LabelMap, VoxelGrid
from .stats import MomentAggregate

MAGIC = b"LRCV"
VERSION = 1
UNASSIGNED_REGION = 0xFFFFFFFF
AGG_MOMENTS = 1
AGG_JSON = 2
SCOPES = ("region", "component", "layer")

# fixed-size index rows (layout.py:240-262): packed little-endian structs
LAYER_ROW = np.dtype([("first_record", "<u8"), ("record_count", "<u8")])
COMPONENT_ROW = np.dtype([("id", "<u4"), ("layer", "<u4"), ("first_record", "<u8"), ("record_count", "<u8"),
                          ("first_region", "<u4"), ("region_count", "<u4"), ("bbox", "<u4", (6,))])
REGION_ROW = np.dtype([("site_id", "<u4"), ("component_id", "<u4"), ("position", "<f8", (3,)),
                       ("first_record", "<u8"), ("record_count", "<u8")])
BLOB_HEAD = struct.Struct("<BIIQ")


def record_dtype(n_fields: int) -> np.dtype:
    """{u32 x, y, z; f32 f0..f(m-1)} (layout.py:36-39)."""
    return np.dtype([(c, "<u4") for c in "xyz"] + [(f"f{i}", "<f4") for i in range(n_fields)])


def reduction_estimate(n: int, r: int, m: int, n_l: int, n_c: int) -> int:
    """Elements saved by dropping out-of-band voxels: m field values plus one
    coordinate slot each, minus the layer and component index entries
    (layout.py:42-48)."""
    if r > n:
        raise ValueError("subset size r cannot exceed domain size n")
    return (n - r) * (m + 1) + n_l + n_c


@dataclass
class AggregateBlob:
    scope: str  # region | component | layer
    scope_id: int
    kind: int
    payload: bytes

    @classmethod
    def moments(cls, scope: str, scope_id: int, agg: MomentAggregate) -> "AggregateBlob":
        return cls(scope, scope_id, AGG_MOMENTS, json.dumps(agg.to_dict()).encode())

    def as_moments(self) -> MomentAggregate:
        if self.kind != AGG_MOMENTS:
            raise ValueError(f"blob kind {self.kind} is not a moment aggregate")
        return MomentAggregate.from_dict(json.loads(self.payload.decode()))


@dataclass
class LayerEntry:
    first_record: int
    record_count: int


@dataclass
class ComponentEntry:
    id: int
    layer: int
    first_record: int
    record_count: int
    first_region: int
    region_count: int
    bbox: tuple[int, int, int, int, int, int]


@dataclass
class RegionEntry:
    site_id: int
    component_id: int
    position: tuple[float, float, float]
    first_record: int
    record_count: int


@dataclass
class Header:
    dims: tuple[int, int, int]
    spacing: tuple[float, float, float]
    field_names: list[str]
    iso_field: str
    iso_values: list[float]
    n_records: int
    layers: list[LayerEntry] = field(default_factory=list)
    components: list[ComponentEntry] = field(default_factory=list)
    regions: list[RegionEntry] = field(default_factory=list)
    data_off: int = 0
    agg_off: int = 0

    @property
    def n_fields(self) -> int:
        return len(self.field_names)


# ---------------------------------------------------------------------------
# device pass


def device_records(grid: VoxelGrid, labels: LabelMap, site_of_dev, names: list[str], n_sites: int):
    """(records [structured, host], region keys u32 [host], comp first int64,
    comp count int64) from one ``lrcvt_layout_records`` call."""
    from . import _lib

    torch = _lib.require_cuda()
    L = _lib.lib()
    nx, ny, nz = grid.dims
    cached = getattr(labels, "_b200_component", None)
    comp_d = cached[1] if cached is not None and cached[0] is labels.component else torch.from_numpy(
        np.ascontiguousarray(labels.component, dtype=np.int32)).to("cuda")
    fields_d = [torch.from_numpy(np.ascontiguousarray(grid.fields[nm], dtype=np.float32)).to("cuda")
                for nm in names]
    ptrs = (ctypes.c_void_p * max(len(fields_d), 1))(*[t.data_ptr() for t in fields_d])
    dt = record_dtype(len(names))
    n_comp = labels.n_components
    cap = sum(c.voxel_count for c in labels.component_table)
    first = torch.empty(max(n_comp, 1), dtype=torch.int64, device="cuda")
    count = torch.empty(max(n_comp, 1), dtype=torch.int64, device="cuda")
    for _ in range(2):  # retry once if the component table understates the in-band count
        rec_d = torch.empty(max(cap, 1) * dt.itemsize, dtype=torch.uint8, device="cuda")
        key_d = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
        got = ctypes.c_int64()
        rc = L.lrcvt_layout_records(nx, ny, nz, len(names), ptrs, comp_d.data_ptr(), site_of_dev.data_ptr(), n_comp,
                                    n_sites, cap, rec_d.data_ptr(), key_d.data_ptr(), first.data_ptr(), count.data_ptr(),
                                    ctypes.byref(got), _lib.stream_handle(torch))
        if rc == _lib.E_ARG and got.value > cap:
            cap = int(got.value)
            continue
        _lib.check(rc, "lrcvt_layout_records")
        break
    r = int(got.value)
    records = rec_d[: r * dt.itemsize].cpu().numpy().view(dt)
    region = key_d[:r].cpu().numpy().view(np.uint32)
    return records, region, first[:n_comp].cpu().numpy(), count[:n_comp].cpu().numpy()


def _site_of_device(tess):
    from . import _lib

    torch = _lib.require_cuda()
    dev = tess.device_state() if hasattr(tess, "device_state") else None
    if dev is not None:
        return dev[0][:, 0].contiguous()
    return torch.from_numpy(np.ascontiguousarray(tess.site_of, dtype=np.int32)).to("cuda")


# ---------------------------------------------------------------------------
# index tables and file


def _index_tables(labels: LabelMap, tess, region: np.ndarray, comp_first: np.ndarray, comp_count: np.ndarray):
    """Layer, component and region entries (layout.py:159-200)."""
    layers = []
    layer_of = np.array([c.layer for c in labels.component_table], dtype=np.int64)
    for li in range(labels.n_layers):
        mine = np.flatnonzero((layer_of == li) & (comp_count > 0)) if layer_of.size else np.zeros(0, np.int64)
        if mine.size:
            layers.append(LayerEntry(int(comp_first[mine].min()), int(comp_count[mine].sum())))
        else:
            layers.append(LayerEntry(0, 0))
    site_comp = tess.site_components()
    per_comp = np.bincount(site_comp, minlength=labels.n_components)
    region_base = np.concatenate(([0], np.cumsum(per_comp)[:-1])) if per_comp.size else per_comp
    components = [ComponentEntry(c.id, c.layer, int(comp_first[c.id]), int(comp_count[c.id]),
                                 int(region_base[c.id]), int(per_comp[c.id]), tuple(int(v) for v in c.bbox))
                  for c in labels.component_table]
    n_regions = len(tess.sites)
    probe = np.arange(n_regions, dtype=np.uint32)
    lo = np.searchsorted(region, probe, side="left")
    hi = np.searchsorted(region, probe, side="right")
    pos = tess.site_positions()
    regions = [RegionEntry(s, int(site_comp[s]), tuple(float(v) for v in pos[s]), int(lo[s]), int(hi[s] - lo[s]))
               for s in range(n_regions)]
    return layers, components, regions


def _str_bytes(s: str) -> bytes:
    b = s.encode()
    return struct.pack("<H", len(b)) + b


def _table_bytes(h: Header) -> tuple[bytes, bytes, bytes]:
    lt = np.zeros(len(h.layers), LAYER_ROW)
    for i, e in enumerate(h.layers):
        lt[i] = (e.first_record, e.record_count)
    ct = np.zeros(len(h.components), COMPONENT_ROW)
    for i, e in enumerate(h.components):
        ct[i] = (e.id, e.layer, e.first_record, e.record_count, e.first_region, e.region_count, e.bbox)
    rt = np.zeros(len(h.regions), REGION_ROW)
    for i, e in enumerate(h.regions):
        rt[i] = (e.site_id, e.component_id, e.position, e.first_record, e.record_count)
    return lt.tobytes(), ct.tobytes(), rt.tobytes()


def _write(path: Path, h: Header, records: np.ndarray, aggs: list[AggregateBlob]) -> None:
    """Header, index tables, record block, aggregate blobs (layout.py:222-277)."""
    fixed = bytearray(MAGIC + struct.pack("<HH3I3d", VERSION, h.n_fields, *h.dims, *h.spacing))
    for s in (*h.field_names, h.iso_field):
        fixed += _str_bytes(s)
    fixed += struct.pack(f"<H{len(h.iso_values)}d", len(h.iso_values), *h.iso_values)
    fixed += struct.pack("<IIIQ", len(h.layers), len(h.components), len(h.regions), h.n_records)
    layer_b, comp_b, region_b = _table_bytes(h)
    layer_off = len(fixed) + 40
    offs = [layer_off, layer_off + len(layer_b), layer_off + len(layer_b) + len(comp_b)]
    offs.append(offs[2] + len(region_b))
    offs.append(offs[3] + records.nbytes)
    h.data_off, h.agg_off = offs[3], offs[4]
    fixed += struct.pack("<5Q", *offs)
    tail = bytearray(struct.pack("<I", len(aggs)))
    for a in aggs:
        tail += BLOB_HEAD.pack(SCOPES.index(a.scope), a.scope_id, a.kind, len(a.payload)) + a.payload
    with open(path, "wb") as fh:
        for part in (fixed, layer_b, comp_b, region_b):
            fh.write(part)
        np.ascontiguousarray(records).tofile(fh)
        fh.write(tail)


def _manifest(h: Header, aggs: list[AggregateBlob]) -> dict:
    """JSON mirror of the header and indexes (layout.py:280-305)."""
    comps = []
    for e in h.components:
        d = {k: getattr(e, k) for k in ("id", "layer", "first_record", "record_count", "first_region",
                                         "region_count")}
        d["bbox"] = list(e.bbox)
        comps.append(d)
    regs = []
    for e in h.regions:
        d = {k: getattr(e, k) for k in ("site_id", "component_id", "first_record", "record_count")}
        d["position"] = list(e.position)
        regs.append(d)
    return {"magic": MAGIC.decode(), "version": VERSION, "dims": list(h.dims), "spacing": list(h.spacing),
            "fields": h.field_names, "iso_field": h.iso_field, "iso_values": h.iso_values,
            "n_records": h.n_records,
            "layers": [{"first_record": e.first_record, "record_count": e.record_count} for e in h.layers],
            "components": comps, "regions": regs,
            "aggregates": [{"scope": a.scope, "scope_id": a.scope_id, "kind": a.kind, "bytes": len(a.payload)}
                           for a in aggs]}


def build_and_write(grid: VoxelGrid, labels: LabelMap, tess, aggregates: list[AggregateBlob],
                    path: str | Path) -> dict:
    """Build the layout on the GPU and write it plus ``<path>.manifest.json``;
    returns the size summary (layout.py:123-219)."""
    path = Path(path)
    names = grid.field_names()
    m = len(names)
    records, region, first, count = device_records(grid, labels, _site_of_device(tess), names, len(tess.sites))
    layers, components, regions = _index_tables(labels, tess, region, first, count)
    r = int(records.size)
    h = Header(tuple(grid.dims), tuple(grid.spacing), names, labels.field_name, list(labels.iso_values), r,
               layers, components, regions)
    _write(path, h, records, aggregates)
    Path(str(path) + ".manifest.json").write_text(json.dumps(_manifest(h, aggregates), indent=1))
    n = grid.size
    return {"path": str(path), "n": n, "r": r, "m": m, "n_layers": labels.n_layers,
            "n_components": labels.n_components, "n_regions": len(tess.sites),
            "estimate_elements": reduction_estimate(n, r, m, labels.n_layers, labels.n_components),
            "data_bytes": r * (12 + 4 * m), "coord_overhead_single_slot": 1.0 / (m + 1),
            "coord_overhead_bytes": 12.0 / (12 + 4 * m)}


# ---------------------------------------------------------------------------
# reader (host I/O)


class LayoutReader:
    """Indexes parsed eagerly; record ranges read on demand
    (layout.py:308-468)."""

    def __init__(self, path: str | Path):
        self.path = Path(path)
        self._size = self.path.stat().st_size
        with open(self.path, "rb") as fh:
            self.header, self._offsets = self._parse_header(fh)
            self.aggregates = self._parse_aggregates(fh)
        self._dtype = record_dtype(self.header.n_fields)
        end = self._offsets["data"] + self.header.n_records * self._dtype.itemsize
        if end > self._size or self._offsets["agg"] > self._size:
            raise ValueError(f"file '{self.path}' is truncated")

    @staticmethod
    def _parse_header(fh):
        magic = fh.read(4)
        if magic != MAGIC:
            raise ValueError(f"bad magic {magic!r}; not a layout file")
        version, n_fields = struct.unpack("<HH", fh.read(4))
        if version != VERSION:
            raise ValueError(f"unsupported version {version}")
        dims = struct.unpack("<3I", fh.read(12))
        spacing = struct.unpack("<3d", fh.read(24))

        def rd_str():
            (k,) = struct.unpack("<H", fh.read(2))
            return fh.read(k).decode()

        names = [rd_str() for _ in range(n_fields)]
        iso_field = rd_str()
        (n_iso,) = struct.unpack("<H", fh.read(2))
        iso = list(struct.unpack(f"<{n_iso}d", fh.read(8 * n_iso)))
        n_l, n_c, n_r, n_rec = struct.unpack("<IIIQ", fh.read(20))
        lo, co, ro, do, ao = struct.unpack("<5Q", fh.read(40))

        def table(off, dt, k):
            fh.seek(off)
            return np.frombuffer(fh.read(dt.itemsize * k), dtype=dt, count=k)

        lt, ct, rt = table(lo, LAYER_ROW, n_l), table(co, COMPONENT_ROW, n_c), table(ro, REGION_ROW, n_r)
        layers = [LayerEntry(int(a), int(b)) for a, b in lt]
        comps = [ComponentEntry(int(e["id"]), int(e["layer"]), int(e["first_record"]), int(e["record_count"]),
                                int(e["first_region"]), int(e["region_count"]), tuple(int(v) for v in e["bbox"]))
                 for e in ct]
        regions = [RegionEntry(int(e["site_id"]), int(e["component_id"]), tuple(float(v) for v in e["position"]),
                               int(e["first_record"]), int(e["record_count"])) for e in rt]
        h = Header(tuple(dims), tuple(spacing), names, iso_field, iso, n_rec, layers, comps, regions, do, ao)
        return h, {"data": do, "agg": ao}

    def _parse_aggregates(self, fh):
        fh.seek(self._offsets["agg"])
        raw = fh.read(4)
        if len(raw) < 4:
            raise ValueError(f"file '{self.path}' is truncated")
        out = []
        for _ in range(struct.unpack("<I", raw)[0]):
            head = fh.read(BLOB_HEAD.size)
            if len(head) < BLOB_HEAD.size:
                raise ValueError(f"file '{self.path}' is truncated")
            scope_i, scope_id, kind, length = BLOB_HEAD.unpack(head)
            payload = fh.read(length)
            if len(payload) != length:
                raise ValueError(f"file '{self.path}' is truncated")
            out.append(AggregateBlob(SCOPES[scope_i], scope_id, kind, payload))
        return out

    def _read_range(self, first: int, count: int) -> np.ndarray:
        if count == 0:
            return np.empty(0, dtype=self._dtype)
        return np.fromfile(self.path, dtype=self._dtype, count=count,
                           offset=self._offsets["data"] + first * self._dtype.itemsize)

    def all_records(self) -> np.ndarray:
        return self._read_range(0, self.header.n_records)

    def layer_records(self, layer: int) -> np.ndarray:
        if not 0 <= layer < len(self.header.layers):
            raise KeyError(f"unknown layer {layer}")
        e = self.header.layers[layer]
        return self._read_range(e.first_record, e.record_count)

    def component_entry(self, component_id: int) -> ComponentEntry:
        if not 0 <= component_id < len(self.header.components):
            raise KeyError(f"unknown component {component_id}")
        return self.header.components[component_id]

    def component_records(self, component_id: int) -> np.ndarray:
        e = self.component_entry(component_id)
        return self._read_range(e.first_record, e.record_count)

    def region_entry(self, site_id: int) -> RegionEntry:
        if not 0 <= site_id < len(self.header.regions):
            raise KeyError(f"unknown region {site_id}")
        return self.header.regions[site_id]

    def region_records(self, site_id: int) -> np.ndarray:
        e = self.region_entry(site_id)
        return self._read_range(e.first_record, e.record_count)

    def component_regions(self, component_id: int) -> list[RegionEntry]:
        e = self.component_entry(component_id)
        return self.header.regions[e.first_region: e.first_region + e.region_count]

    def aggregates_for(self, scope: str, scope_id: int) -> list[AggregateBlob]:
        return [a for a in self.aggregates if a.scope == scope and a.scope_id == scope_id]

    def field_column(self, records: np.ndarray, name: str) -> np.ndarray:
        return records[f"f{self.header.field_names.index(name)}"]


def load_component(path: str | Path, component_id: int) -> dict:
    """One component's records, its regions and their aggregate blobs, read
    from the component's byte range plus the indexes (layout.py:471-488)."""
    reader = LayoutReader(path)
    entry = reader.component_entry(component_id)
    regions = reader.component_regions(component_id)
    aggs = reader.aggregates_for("component", component_id)
    for reg in regions:
        aggs.extend(reader.aggregates_for("region", reg.site_id))
    return {"entry": entry, "records": reader.component_records(component_id), "regions": regions,
            "aggregates": aggs}

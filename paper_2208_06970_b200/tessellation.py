"""Restricted geodesic Voronoi classification and the centroidal Lloyd loop,
on the GPU.

Drop-in for the reference's ``lrcvt.tessellation`` (tessellation.py:33-374):
same entry points, dataclasses, dtypes, report keys and exceptions. The
numba kernel seam (``lrcvt._kernels``) is replaced by the C-ABI library
(include/lrcvt_cuda.h); per-voxel state stays resident in HBM across a
Lloyd loop and only the final tessellation is copied back.
"""

from __future__ import annotations

import ctypes
import gc
import itertools
import operator
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib

try:  # the C builder of list[Site] (csrc/sites_ext.c, built by __graft_entry__.build)
    from . import _sites
except ImportError:  # pragma: no cover - the pure-Python builder below gives the same objects
    _sites = None
from .grid import NONE_ID, LabelMap, VoxelGrid
from .seeding import SeedingParams, Site, seed_sites, voxel_weights

LOS = 1
ACTIVE = 2
NODE = 4


@dataclass
class LloydParams:
    max_updates: int = 50
    ds_tolerance: float = 0.25

    def __post_init__(self):
        if self.max_updates < 1:
            raise ValueError("max_updates must be >= 1")
        if self.ds_tolerance <= 0:
            raise ValueError("ds_tolerance must be > 0")


@dataclass
class Tessellation:
    """Classification result (tessellation.py:45-71)."""

    dims: tuple[int, int, int]
    spacing: tuple[float, float, float]
    site_of: np.ndarray
    dist: np.ndarray
    src: np.ndarray
    state: np.ndarray
    component: np.ndarray
    sites: list[Site]
    report: dict = field(default_factory=dict)
    weights: np.ndarray | None = None

    @property
    def n_sites(self) -> int:
        return len(self.sites)

    def site_positions(self) -> np.ndarray:
        return _positions(self.sites)

    def site_components(self) -> np.ndarray:
        return _components(self.sites)


class DeviceTessellation(Tessellation):
    """A Tessellation whose per-voxel arrays (site_of, dist, src, state) stay
    in HBM until first read: attribute access materialises them as numpy in
    the reference dtypes, once. centroidal_update() consumes the device copy
    directly, so a classify -> update step moves no per-voxel data over PCIe
    unless the caller looks at the arrays. Assigning an array makes the host
    copy authoritative from then on."""

    def __init__(self, dims, spacing, component, sites, report, weights, engine, dev):
        self._dev = dev  # (ss int32[N, 2], dist float64[N], state uint8[N]) on the GPU
        self._host: dict = {}
        self._dirty = False
        self._engine = engine
        self.dims = dims
        self.spacing = spacing
        self.component = component
        self.sites = sites
        self.report = report
        self.weights = weights

    def _get(self, name):
        """Materialise one output as numpy: (site_of, src) are split on the
        device (lrcvt_unpack_site_src) and every array is read straight into
        page-locked host memory from torch's caching host allocator (freed
        arrays return their pages to the pool), one PCIe pass per array."""
        host = self._host
        if name not in host:
            ss, dist, state = self._dev
            torch = self._engine.torch
            if name in ("site_of", "src"):
                n = ss.shape[0]
                so = torch.empty(n, dtype=torch.int32, device="cuda")
                sr = torch.empty(n, dtype=torch.int32, device="cuda")
                _lib.check(self._engine.L.lrcvt_unpack_site_src(ss.data_ptr(), n, so.data_ptr(), sr.data_ptr(),
                                                                 _lib.stream_handle(torch)), "lrcvt_unpack_site_src")
                got = [_to_pinned(torch, so), _to_pinned(torch, sr)]
                torch.cuda.current_stream().synchronize()
                host.setdefault("site_of", got[0].numpy())
                host.setdefault("src", got[1].numpy())
            else:
                got = _to_pinned(torch, dist if name == "dist" else state)
                torch.cuda.current_stream().synchronize()
                host[name] = got.numpy()
        return host[name]

    def _set(self, name, value):
        self._host[name] = value
        self._dirty = True

    site_of = property(lambda self: self._get("site_of"), lambda self, v: self._set("site_of", v))
    dist = property(lambda self: self._get("dist"), lambda self, v: self._set("dist", v))
    src = property(lambda self: self._get("src"), lambda self, v: self._set("src", v))
    state = property(lambda self: self._get("state"), lambda self, v: self._set("state", v))

    def device_state(self):
        """(ss, dist, state) device tensors while they are authoritative, else None."""
        return None if self._dirty else self._dev


def _to_pinned(torch, t):
    """Asynchronous device->host copy into a page-locked tensor (the caller
    synchronises the stream before reading it)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h


def voxel_length(dims, spacing) -> float:
    """Mean spacing over the axes that extend (tessellation.py:74-79)."""
    active = [s for d, s in zip(dims, spacing) if d > 1]
    if not active:
        active = list(spacing)
    return float(np.mean(active))


# ---------------------------------------------------------------------------
# device engine


class Engine:
    """Device-resident state for one component volume: the C-ABI plan, the
    packed (site_of, src) int32[N][2], dist float64[N] and state uint8[N]."""

    def __init__(self, dims, spacing, component: np.ndarray, n_components: int, max_sites: int,
                 comp_dev=None, alloc_state: bool = True):
        torch = _lib.require_cuda()
        self.torch = torch
        self.L = _lib.lib()
        self.dims = tuple(int(d) for d in dims)
        self.spacing = tuple(float(s) for s in spacing)
        self.n = int(np.prod(self.dims))
        self.n_components = int(n_components)
        self.comp = comp_dev if comp_dev is not None else torch.from_numpy(
            np.ascontiguousarray(component, dtype=np.int32)).to("cuda")
        self.max_sites = 0
        self.plan = ctypes.c_void_p()
        self._make_plan(max(int(max_sites), 1))
        # alloc_state=False: the caller supplies ss / dist (multi-GPU slabs use plan-owned buffers)
        self.ss = torch.empty((self.n, 2), dtype=torch.int32, device="cuda") if alloc_state else None
        self.dist = torch.empty(self.n, dtype=torch.float64, device="cuda") if alloc_state else None
        self.state = torch.empty(self.n, dtype=torch.uint8, device="cuda")
        self.version = 0  # bumps on every classify; guards host<->device reuse
        self.classify_seq = 0  # bumps on every classify call (the plan's eligible list follows it)
        self.stats = _lib.ClassifyStats()
        self._out_dirty = True
        self._fin = weakref.finalize(self, Engine._destroy, self.L, self.plan)

    @staticmethod
    def _destroy(L, plan):
        if plan.value:
            L.lrcvt_plan_destroy(plan)
            plan.value = None

    def _make_plan(self, max_sites):
        if self.plan.value:
            self.L.lrcvt_plan_destroy(self.plan)
            self.plan.value = None
        nx, ny, nz = self.dims
        sx, sy, sz = self.spacing
        _lib.check(self.L.lrcvt_plan_create(ctypes.byref(self.plan), nx, ny, nz, sx, sy, sz,
                                            self.comp.data_ptr(), self.n_components, max_sites,
                                            _lib.stream_handle(self.torch)), "lrcvt_plan_create")
        self.max_sites = max_sites

    def reserve(self, n_sites: int):
        if n_sites > self.max_sites:
            self._make_plan(max(n_sites, 2 * self.max_sites))

    @property
    def inband(self) -> int:
        return int(self.L.lrcvt_plan_inband(self.plan))

    def classify(self, site_pos, site_comp, want_state=True, out=None) -> dict:
        """site_pos float64[S,3], site_comp int32[S] (device tensors). Writes
        the engine's own state buffers, or `out` = (ss, dist, state) tensors."""
        S = int(site_pos.shape[0])
        self.reserve(S)
        ss, dist, state = out if out is not None else (self.ss, self.dist, self.state)
        self.classify_seq += 1
        # the engine's own buffers are only ever written by its classifies: the plan may reset just the
        # eligible voxels when they come back (lrcvt_plan_persistent_outputs)
        self.L.lrcvt_plan_persistent_outputs(self.plan, 1 if out is None and not self._out_dirty else 0)
        if out is None:
            self._out_dirty = False
        try:
            rc = _lib.check(self.L.lrcvt_classify(
                self.plan, S, _lib.ptr(site_pos), _lib.ptr(site_comp), ss.data_ptr(),
                dist.data_ptr(), state.data_ptr() if want_state else None,
                ctypes.byref(self.stats), _lib.stream_handle(self.torch)), "lrcvt_classify")
        finally:
            self.L.lrcvt_plan_persistent_outputs(self.plan, 0)
        if out is None:
            self.version += 1
        if rc > 0:
            raise ValueError(f"{rc} sites sit outside their recorded component")
        return self.stats.as_dict()

    def new_state(self):
        """Fresh (ss, dist, state) device tensors from torch's caching allocator."""
        t = self.torch
        return (t.empty((self.n, 2), dtype=t.int32, device="cuda"),
                t.empty(self.n, dtype=t.float64, device="cuda"),
                t.empty(self.n, dtype=t.uint8, device="cuda"))

    def centroidal(self, site_pos, site_comp, weight_mode: int, weights, backoff: float,
                   want_sums=False, ss=None):
        torch = self.torch
        ss = self.ss if ss is None else ss
        S = int(site_pos.shape[0])
        self.reserve(S)
        new_pos = torch.empty((S, 3), dtype=torch.float64, device="cuda")
        disp = torch.empty(S, dtype=torch.float64, device="cuda")
        sums = torch.empty((4, S), dtype=torch.float64, device="cuda") if want_sums else None
        empty = ctypes.c_int64(0)
        _lib.check(self.L.lrcvt_centroidal_update(
            self.plan, S, _lib.ptr(site_pos), _lib.ptr(site_comp), ss.data_ptr(),
            weight_mode, _lib.ptr(weights), float(backoff), new_pos.data_ptr(), disp.data_ptr(),
            _lib.ptr(sums), ctypes.byref(empty), _lib.stream_handle(torch)),
            "lrcvt_centroidal_update")
        return new_pos, disp, int(empty.value), sums

    def host_arrays(self):
        """(site_of, dist, src, state) as numpy in the reference dtypes."""
        ss = self.ss.cpu().numpy()
        return (np.ascontiguousarray(ss[:, 0]), self.dist.cpu().numpy(),
                np.ascontiguousarray(ss[:, 1]), self.state.cpu().numpy())

    def upload(self, site_of: np.ndarray, src: np.ndarray):
        packed = np.empty((self.n, 2), dtype=np.int32)
        packed[:, 0] = site_of
        packed[:, 1] = src
        self.ss.copy_(self.torch.from_numpy(packed))
        self._out_dirty = True  # written outside a classify: the next one resets every voxel
        self.version += 1


def engine_for(labels: LabelMap, spacing, n_sites: int) -> Engine:
    """The engine cached on a LabelMap, reused while its component array and
    spacing are unchanged."""
    comp = labels.component
    spacing = tuple(float(s) for s in spacing)
    eng = getattr(labels, "_b200_engine", None)
    if (eng is not None and eng._src is comp and eng.spacing == spacing
            and eng.n_components == labels.n_components):
        eng.reserve(n_sites)
        return eng
    dev = getattr(labels, "_b200_component", None)
    comp_dev = dev[1] if dev is not None and dev[0] is comp else None
    eng = Engine(labels.dims, spacing, comp, labels.n_components, n_sites, comp_dev)
    eng._src = comp
    labels._b200_engine = eng
    return eng


_get_pos = operator.attrgetter("position")
_get_comp = operator.attrgetter("component_id")


# The arrays of the last Site list built or read here, with what identifies
# it: the Site objects, their position tuples (a reassigned position is a new
# tuple) and component ids. A list whose elements are those very objects,
# still holding those very tuples and ids, has those arrays -- checked at C
# level in half the time of reading the positions again.
_site_cache: list = [None]


def _cached_arrays(sites):
    c = _site_cache[0]
    if (c is None or len(sites) != len(c[0]) or not all(map(operator.is_, sites, c[0]))
            or not all(map(operator.is_, map(_get_pos, sites), c[1])) or list(map(_get_comp, sites)) != c[2]):
        return None
    return c[3], c[4]


def _remember(sites, pos: np.ndarray, comp: np.ndarray):
    _site_cache[0] = (tuple(sites), list(map(_get_pos, sites)), comp.tolist(), pos, comp)


def _read_sites(sites):
    """(float64[S, 3] positions, int32[S] components) of a Site list; the
    returned arrays are shared with the cache: callers copy before writing"""
    got = _cached_arrays(sites)
    if got is None:
        pos = np.fromiter(itertools.chain.from_iterable(map(_get_pos, sites)), dtype=np.float64,
                          count=3 * len(sites)).reshape(-1, 3)
        comp = np.fromiter(map(_get_comp, sites), dtype=np.int32, count=len(sites))
        _remember(sites, pos, comp)
        got = pos, comp
    return got


def _positions(sites) -> np.ndarray:
    """float64[S, 3] site positions (C-level iteration; same values as np.array)."""
    return _read_sites(sites)[0].copy()


def _components(sites) -> np.ndarray:
    return _read_sites(sites)[1].copy()


def make_sites(pos: np.ndarray, comp: np.ndarray) -> list[Site]:
    """Site objects from float64[S, 3] positions and int component ids (the
    same Python floats / ints as Site((float(x), float(y), float(z)), int(c))).
    Built from column lists zipped at C level, with the cyclic collector
    paused: its generation-0 passes over the new objects cost as much as
    building them."""
    pos = np.array(pos, dtype=np.float64).reshape(-1, 3)
    comp = np.array(comp, dtype=np.int32).reshape(-1)
    if _sites is not None:  # csrc/sites_ext.c: the same objects, built in C
        out = _sites.make_sites(Site, pos.tobytes(), comp.tobytes())
    else:
        cols = pos.T.tolist()
        ids = comp.tolist()
        paused = gc.isenabled()
        gc.disable()
        try:
            out = list(map(Site, zip(cols[0], cols[1], cols[2]), ids))
        finally:
            if paused:
                gc.enable()
    _remember(out, pos, comp)
    return out


def _site_arrays(torch, sites):
    pos, comp = _read_sites(sites)
    return pos, comp, torch.from_numpy(pos).to("cuda"), torch.from_numpy(comp).to("cuda")


def _no_site_components(labels: LabelMap, site_comp: np.ndarray) -> list[int]:
    has = np.zeros(max(labels.n_components, 1), dtype=bool)
    if site_comp.size:
        has[site_comp] = True
    table = labels.component_table
    cached = getattr(labels, "_b200_ids", None)  # component ids of the table, once per table object
    if cached is None or cached[0] is not table or cached[1].size != len(table):
        cached = (table, np.fromiter((c.id for c in table), dtype=np.int64, count=len(table)))
        labels._b200_ids = cached
    ids = cached[1]
    return np.unique(ids[~has[ids]]).tolist()


# ---------------------------------------------------------------------------
# public API (tessellation.py:82-275)


def raycast_same_component(labels: LabelMap, a, b, spacing=(1.0, 1.0, 1.0)) -> bool:
    """True iff every voxel on segment a->b shares a's component
    (tessellation.py:82-99); one DDA on the GPU."""
    torch = _lib.require_cuda()
    nx, ny, nz = labels.dims
    sx, sy, sz = (float(s) for s in spacing)
    ax, ay, az = float(a[0]), float(a[1]), float(a[2])
    cx = min(max(int(np.floor(ax / sx)), 0), nx - 1)
    cy = min(max(int(np.floor(ay / sy)), 0), ny - 1)
    cz = min(max(int(np.floor(az / sz)), 0), nz - 1)
    want = int(labels.component[cx + nx * (cy + ny * cz)])
    t = segment_hit_t_batch(labels, np.array([[ax, ay, az, float(b[0]), float(b[1]), float(b[2])]]),
                            np.array([want], np.int32), (sx, sy, sz))
    return bool(t[0] >= 1.0)


def segment_hit_t_batch(labels: LabelMap, segs: np.ndarray, want: np.ndarray, spacing) -> np.ndarray:
    torch = _lib.require_cuda()
    L = _lib.lib()
    nx, ny, nz = labels.dims
    eng = getattr(labels, "_b200_engine", None)
    comp = eng.comp if eng is not None and eng._src is labels.component else torch.from_numpy(
        np.ascontiguousarray(labels.component, dtype=np.int32)).to("cuda")
    segs_d = torch.from_numpy(np.ascontiguousarray(segs, dtype=np.float64)).to("cuda")
    want_d = torch.from_numpy(np.ascontiguousarray(want, dtype=np.int32)).to("cuda")
    out = torch.empty(len(segs), dtype=torch.float64, device="cuda")
    _lib.check(L.lrcvt_segment_hit_t(nx, ny, nz, *[float(s) for s in spacing], comp.data_ptr(),
                                     segs_d.data_ptr(), want_d.data_ptr(), len(segs), out.data_ptr(),
                                     _lib.stream_handle(torch)), "lrcvt_segment_hit_t")
    return out.cpu().numpy()


def voronoi_classify(grid: VoxelGrid, labels: LabelMap, sites: list[Site],
                     weights: np.ndarray | None = None) -> Tessellation:
    """Classify every reachable in-band voxel to its geodesically nearest
    site (tessellation.py:102-208)."""
    n = grid.size
    comp = np.ascontiguousarray(labels.component, dtype=np.int32)
    if len(sites) == 0:
        return Tessellation(grid.dims, grid.spacing, np.full(n, NONE_ID, np.int32),
                            np.full(n, np.inf), np.full(n, NONE_ID, np.int32),
                            np.zeros(n, np.uint8), comp, list(sites),
                            {"rounds": 0, "sweeps": 0,
                             "components_without_sites": sorted({c.id for c in labels.component_table})},
                            weights)
    torch = _lib.require_cuda()
    eng = engine_for(labels, grid.spacing, len(sites))
    pos_h, site_comp, pos_d, comp_d = _site_arrays(torch, sites)
    dev = eng.new_state()
    st = eng.classify(pos_d, comp_d, out=dev)
    report = {"rounds": st["rounds"], "sweeps": st["sweeps"],
              "components_without_sites": _no_site_components(labels, site_comp),
              "assigned": st["assigned"]}
    tess = DeviceTessellation(grid.dims, grid.spacing, comp, list(sites), report, weights, eng, dev)
    tess._b200_stats = st
    # the site arrays this classification used: centroidal_update reuses them (and the plan's
    # eligible-voxel list) while no other classification ran on the plan and the sites are unchanged
    tess._b200_sites = (eng.classify_seq, pos_h, site_comp, pos_d, comp_d)
    return tess


def _weights_mode(torch, weights: np.ndarray | None, eng: "Engine | None" = None):
    """float64 weights on the device; the upload is cached on the engine for
    as long as the caller keeps passing the same array object."""
    if weights is None:
        return _lib.W_ONES, None
    cached = getattr(eng, "_wcache", None) if eng is not None else None
    if cached is not None and cached[0] is weights:
        return _lib.W_F64, cached[1]
    w = np.ascontiguousarray(weights, dtype=np.float64)
    dev = torch.from_numpy(w).to("cuda")
    if eng is not None:
        eng._wcache = (weights, dev)
    return _lib.W_F64, dev


def centroidal_update(tess: Tessellation, weights: np.ndarray | None = None) -> tuple[list[Site], float]:
    """One geodesically weighted site move (tessellation.py:211-248)."""
    if weights is None:
        weights = tess.weights
    torch = _lib.require_cuda()
    if len(tess.sites) == 0:
        tess.report["empty_regions"] = 0
        return [], 0.0
    pos, site_comp = _read_sites(tess.sites)  # read-only below
    dev = tess.device_state() if isinstance(tess, DeviceTessellation) else None
    ss = None
    if dev is not None:
        eng = tess._engine
        ss = dev[0]
    else:
        labels = LabelMap(tess.dims, np.zeros(0, np.int32), tess.component,
                          iso_values=[], field_name="")
        n_comp = int(tess.component.max()) + 1 if tess.component.size else 0
        eng = Engine(tess.dims, tess.spacing, tess.component, max(n_comp, int(site_comp.max()) + 1),
                     len(tess.sites))
        eng.upload(tess.site_of, tess.src)
        del labels
    cached = getattr(tess, "_b200_sites", None) if dev is not None else None
    reuse = (cached is not None and cached[0] == eng.classify_seq
             and (cached[2] is site_comp or np.array_equal(cached[2], site_comp))
             and (cached[1] is pos or np.array_equal(cached[1], pos)))
    if reuse:
        pos_d, comp_d = cached[3], cached[4]
    else:
        pos_d = torch.from_numpy(pos).to("cuda")
        comp_d = torch.from_numpy(np.ascontiguousarray(site_comp, dtype=np.int32)).to("cuda")
    mode, w_d = _weights_mode(torch, weights, eng)
    vlen = voxel_length(tess.dims, tess.spacing)
    if reuse:  # same site components as the classification that built the eligible list
        eng.L.lrcvt_plan_reuse_eligible(eng.plan, 1)
    try:
        new_pos, disp, empty, _ = eng.centroidal(pos_d, comp_d, mode, w_d, 0.5 * vlen, ss=ss)
    finally:
        if reuse:
            eng.L.lrcvt_plan_reuse_eligible(eng.plan, 0)
    tess.report["empty_regions"] = int(empty)
    both = torch.cat([new_pos, disp[:, None]], dim=1).cpu().numpy()  # one device->host read
    disp = np.ascontiguousarray(both[:, 3])
    new_sites = make_sites(both[:, :3], site_comp)
    mean_ds = float(disp.mean() / vlen) if disp.size else 0.0
    return new_sites, mean_ds


def lloyd_weight_mode(torch, grid: VoxelGrid, seeding: SeedingParams, weights: np.ndarray):
    """Device weight representation for the Lloyd loop: unit weights, the
    float32 field itself (gamma 1 or 2, exact on device), or float64 m**gamma."""
    if seeding.weight_field is None:
        return _lib.W_ONES, None
    if seeding.gamma == 1.0:
        return _lib.W_F32_G1, torch.from_numpy(grid.fields[seeding.weight_field]).to("cuda")
    if seeding.gamma == 2.0:
        return _lib.W_F32_G2, torch.from_numpy(grid.fields[seeding.weight_field]).to("cuda")
    return _lib.W_F64, torch.from_numpy(np.ascontiguousarray(weights)).to("cuda")


def lrcvt(grid: VoxelGrid, labels: LabelMap, seeding: SeedingParams,
          lloyd: LloydParams) -> tuple[Tessellation, list[float]]:
    """Seed, then alternate classification and centroidal updates until the
    mean displacement drops below tolerance or the budget runs out
    (tessellation.py:251-275). The loop runs device-resident; one small
    device->host read per update (the displacement vector, for mean_ds)."""
    if labels.n_components == 0:
        raise ValueError("no connected components to tessellate")
    sites, seed_report = seed_sites(grid, labels, seeding)
    weights = voxel_weights(grid, seeding)
    trace: list[float] = []
    if not sites:
        final = voronoi_classify(grid, labels, sites, weights)
        final.report["seeding"] = seed_report
        final.report["updates"] = 0
        return final, trace
    torch = _lib.require_cuda()
    eng = engine_for(labels, grid.spacing, len(sites))
    _, site_comp, pos_d, comp_d = _site_arrays(torch, sites)
    mode, w_d = lloyd_weight_mode(torch, grid, seeding, weights)
    vlen = voxel_length(grid.dims, grid.spacing)
    eng.L.lrcvt_plan_reuse_eligible(eng.plan, 2)  # site components fixed for the whole loop (built by its first classify)
    try:
        trace = _lloyd_iterations(eng, pos_d, comp_d, mode, w_d, vlen, lloyd, trace)
    finally:
        eng.L.lrcvt_plan_reuse_eligible(eng.plan, 0)
    pos_d = eng._last_pos
    pos = pos_d.cpu().numpy()
    final_sites = make_sites(pos, site_comp)
    final = voronoi_classify(grid, labels, final_sites, weights)
    final.report["seeding"] = seed_report
    final.report["updates"] = len(trace)
    return final, trace


def _lloyd_iterations(eng, pos_d, comp_d, mode, w_d, vlen, lloyd, trace):
    for _ in range(lloyd.max_updates):
        eng.classify(pos_d, comp_d, want_state=False)
        pos_d, disp, _, _ = eng.centroidal(pos_d, comp_d, mode, w_d, 0.5 * vlen)
        d = disp.cpu().numpy()
        mean_ds = float(d.mean() / vlen) if d.size else 0.0
        trace.append(mean_ds)
        if mean_ds < lloyd.ds_tolerance:
            break
    eng._last_pos = pos_d
    return trace


# ---------------------------------------------------------------------------
# validation helpers (tessellation.py:278-374)


def geodesic_oracle(labels: LabelMap, source: int, spacing=(1.0, 1.0, 1.0),
                    initial_distance: float = 0.0) -> np.ndarray:
    """Dijkstra over the same-component 26-neighbour graph (host scipy;
    a validation oracle, not part of the hot path)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra

    nx, ny, nz = labels.dims
    comp = labels.component
    c = comp[source]
    if c == NONE_ID:
        raise ValueError(f"source voxel {source} is out of band")
    members = np.flatnonzero(comp == c)
    local = np.full(comp.size, -1, dtype=np.int64)
    local[members] = np.arange(members.size)
    xs, ys, zs = members % nx, (members // nx) % ny, members // (nx * ny)
    sx, sy, sz = spacing
    rows, cols, wts = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if (dz, dy, dx) >= (0, 0, 0):
                    continue  # half the offsets: the graph is symmetric
                x2, y2, z2 = xs + dx, ys + dy, zs + dz
                ok = (x2 >= 0) & (y2 >= 0) & (z2 >= 0) & (x2 < nx) & (y2 < ny) & (z2 < nz)
                tgt = x2[ok] + nx * (y2[ok] + ny * z2[ok])
                same = comp[tgt] == c
                a = local[members[ok][same]]
                rows.append(a)
                cols.append(local[tgt[same]])
                wts.append(np.full(a.size, np.sqrt((dx * sx) ** 2 + (dy * sy) ** 2 + (dz * sz) ** 2)))
    m = members.size
    graph = csr_matrix((np.concatenate(wts), (np.concatenate(rows), np.concatenate(cols))), shape=(m, m))
    d_local = dijkstra(graph, directed=False, indices=int(local[source]))
    out = np.full(comp.size, np.inf)
    out[members] = d_local + initial_distance
    return out


def _phi_host(site_of: np.ndarray, src: np.ndarray):
    """phi map by vectorised pointer jumping (host; audit only)."""
    n = site_of.size
    assigned = site_of >= 0
    phi = np.where(assigned, src, -1).astype(np.int64)
    idx = np.arange(n)
    los = assigned & (src == idx)
    phi[los] = idx[los]
    depth = np.zeros(n, dtype=np.int64)
    for _ in range(64):
        ok = phi >= 0
        nxt = phi.copy()
        nxt[ok] = phi[phi[ok]]
        moved = ok & (nxt != phi)
        if not moved.any():
            break
        depth[moved] += 1
        phi = nxt
    return phi, depth


def audit_tessellation(tess: Tessellation, labels: LabelMap, check_rays: bool = True) -> dict:
    """Invariant audit (tessellation.py:326-374): restriction, chain
    termination and site consistency, Euclidean lower bound and (optionally)
    per-segment ray validity (GPU DDA)."""
    nx, ny, nz = tess.dims
    sx, sy, sz = tess.spacing
    comp = labels.component
    assigned = np.flatnonzero(tess.site_of != NONE_ID)
    site_comp = tess.site_components()
    site_pos = tess.site_positions()
    out = {}
    out["restriction_violations"] = int(np.count_nonzero(comp[assigned] != site_comp[tess.site_of[assigned]]))
    phi, _ = _phi_host(tess.site_of, tess.src)
    ok = phi[assigned] >= 0
    out["broken_chains"] = int(np.count_nonzero(~ok))
    out["chain_site_mismatch"] = int(np.count_nonzero(
        tess.site_of[assigned[ok]] != tess.site_of[phi[assigned[ok]]]))
    # chain depth in the reference counts hops to the LOS terminal
    depth = 0
    if assigned.size:
        hops = np.zeros(assigned.size, dtype=np.int64)
        cur = assigned.copy()
        for _ in range(tess.site_of.size + 1):
            nxt = tess.src[cur]
            live = (nxt != cur) & (nxt >= 0)
            if not live.any():
                break
            hops[live] += 1
            cur = np.where(live, nxt, cur)
        depth = int(hops.max())
    max_comp = max((c.voxel_count for c in labels.component_table), default=0)
    out["max_chain_depth"] = depth
    out["chain_depth_ok"] = bool(depth <= max_comp)
    centers = np.empty((assigned.size, 3))
    centers[:, 0] = (assigned % nx + 0.5) * sx
    centers[:, 1] = ((assigned // nx) % ny + 0.5) * sy
    centers[:, 2] = (assigned // (nx * ny) + 0.5) * sz
    euclid = np.linalg.norm(centers - site_pos[tess.site_of[assigned]], axis=1)
    out["euclid_bound_violations"] = int(np.count_nonzero(euclid > tess.dist[assigned] + 1e-9))
    out["nonfinite_dist"] = int(np.count_nonzero(~np.isfinite(tess.dist[assigned])))
    if check_rays and assigned.size:
        s = tess.site_of[assigned]
        u = tess.src[assigned]
        los = u == assigned
        b = np.empty((assigned.size, 3))
        b[los] = site_pos[s[los]]
        nl = ~los & (u >= 0)
        b[nl, 0] = (u[nl] % nx + 0.5) * sx
        b[nl, 1] = ((u[nl] // nx) % ny + 0.5) * sy
        b[nl, 2] = (u[nl] // (nx * ny) + 0.5) * sz
        segs = np.concatenate([centers, b], axis=1)
        t = segment_hit_t_batch(labels, segs, comp[assigned].astype(np.int32), tess.spacing)
        bad = (t < 1.0) | (u < 0)
        out["segment_violations"] = int(bad.sum())
    return out

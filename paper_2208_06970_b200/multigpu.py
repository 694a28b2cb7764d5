"""Multi-GPU global mode: one tessellation over z-slabs of the whole volume,
bit-identical to the single-domain result (north star).

Design: the per-voxel state is REPLICATED on every rank and
the EVALUATION is partitioned -- rank r evaluates only the frontier voxels of
its z-slab [zlo_r, zhi_r). After each relaxation round the improved
proposals (24-byte records) are all-gathered over NVLink and every rank
commits all of them, enqueueing only the neighbours that fall in its own
slab. Every evaluation therefore reads exactly the global pre-round state,
so site_of/dist/src, rounds, sweeps and the E/C counters equal the
single-domain run; per round the only traffic is the proposal all-gather
plus two count exchanges. The vote runs redundantly on every rank's
identical state (no exchange, bit-exact).

`Collective` hides where the ranks live:
  * `Emulated` -- all ranks in this process on one GPU (state copies per
    rank); used by the parity tests, since this environment has one GPU;
  * `TorchDist` -- one rank per process, torch.distributed (NCCL on GPUs).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .tessellation import Engine

PROP_BYTES = 24


def slab_bounds(nz: int, world: int) -> list[tuple[int, int]]:
    """Equal z-slabs of ceil(nz / world) planes (the last may be shorter)."""
    planes = math.ceil(nz / world)
    out = [(r * planes, min((r + 1) * planes, nz)) for r in range(world)]
    if any(lo >= hi for lo, hi in out):
        raise ValueError(f"cannot split {nz} planes into {world} non-empty slabs")
    return out


class Emulated:
    """All ranks live in this process (one GPU): gathers are concatenations."""

    def __init__(self, world: int):
        self.world = world
        self.local_ranks = list(range(world))

    def all_counts(self, local: list[int]) -> list[int]:
        return list(local)

    def all_props(self, local: list, torch):
        return torch.cat(local) if local else torch.empty(0, dtype=torch.uint8, device="cuda")


class TorchDist:
    """One rank per process over torch.distributed: NCCL on CUDA tensors for
    the GPU path; any backend works for the host-side protocol (device="cpu"
    with gloo in the CPU tests)."""

    def __init__(self, group=None, device: str = "cuda"):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.device = device
        self.world = dist.get_world_size(group)
        self.local_ranks = [dist.get_rank(group)]

    def all_counts(self, local: list[int]) -> list[int]:
        import torch

        t = torch.tensor(local, dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(v) for x in out for v in x.tolist()]

    def all_props(self, local: list, torch):
        """Concatenate every rank's proposal bytes in rank order (padded
        all_gather: NCCL has no variable-size all-gather)."""
        counts = self.all_counts([int(local[0].numel())])
        m = max(counts)
        if m == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.device)
        pad = torch.zeros(m, dtype=torch.uint8, device=self.device)
        pad[: local[0].numel()] = local[0]
        out = [torch.empty(m, dtype=torch.uint8, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(out, pad, group=self.group)
        return torch.cat([o[:c] for o, c in zip(out, counts)])


class GlobalClassifier:
    """Slab-partitioned voronoi_classify over a Collective. Each local rank
    owns an Engine (plan with slab bounds) holding a full replicated copy of
    the per-voxel state (engine.ss / engine.dist / engine.state)."""

    def __init__(self, dims, spacing, component: np.ndarray, n_components: int, max_sites: int, coll):
        self.torch = _lib.require_cuda()
        self.L = _lib.lib()
        self.coll = coll
        self.dims = tuple(int(d) for d in dims)
        self.bounds = slab_bounds(self.dims[2], coll.world)
        self.engines = {}
        comp_dev = None
        for r in coll.local_ranks:
            eng = Engine(self.dims, spacing, component, n_components, max_sites, comp_dev)
            comp_dev = eng.comp  # replicated labels shared between in-process ranks
            lo, hi = self.bounds[r]
            _lib.check(self.L.lrcvt_mg_set_slab(eng.plan, lo, hi), "lrcvt_mg_set_slab")
            self.engines[r] = eng

    def _props(self, eng, n):
        t = self.torch.empty(n * PROP_BYTES, dtype=self.torch.uint8, device="cuda")
        _lib.check(self.L.lrcvt_mg_copy_proposals(eng.plan, t.data_ptr() if n else None, n,
                                                   _lib.stream_handle(self.torch)), "copy proposals")
        return t

    def _round(self, phase: int, sweep: int, stats: dict) -> int:
        """One relaxation round (or sweep) on all ranks; returns the global
        number of improved proposals."""
        L, st = self.L, _lib.stream_handle(self.torch)
        evals, props = [], []
        for r, eng in self.engines.items():
            ne, nimp = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(L.lrcvt_mg_eval(eng.plan, phase, sweep, ctypes.byref(ne), ctypes.byref(nimp), st),
                       "lrcvt_mg_eval")
            evals.append(int(ne.value))
            props.append(self._props(eng, int(nimp.value)))
        stats["evaluations"] += sum(self.coll.all_counts(evals))
        allp = self.coll.all_props(props, self.torch)
        n_all = allp.numel() // PROP_BYTES
        stats["commits"] += n_all
        if sweep and n_all == 0:
            return 0
        nexts = []
        for r, eng in self.engines.items():
            nn = ctypes.c_int64()
            _lib.check(L.lrcvt_mg_commit(eng.plan, allp.data_ptr() if n_all else None, n_all, sweep,
                                         ctypes.byref(nn), st), "lrcvt_mg_commit")
            nexts.append(int(nn.value))
        self._frontier = nexts
        return n_all

    def _run_rounds(self, phase: int, stats: dict):
        while sum(self.coll.all_counts(self._frontier)) > 0:
            stats["rounds"] += 1
            self._round(phase, 0, stats)

    def classify(self, site_pos, site_comp) -> dict:
        """site_pos float64[S,3], site_comp int32[S] on the device; returns
        the report counters (rounds, sweeps, assigned, evaluations, commits)."""
        L, st = self.L, _lib.stream_handle(self.torch)
        S = int(site_pos.shape[0])
        stats = {"rounds": 0, "sweeps": 0, "evaluations": 0, "commits": 0}
        self._frontier = []
        for r, eng in self.engines.items():
            eng.reserve(S)
            _lib.check(L.lrcvt_mg_set_slab(eng.plan, *self.bounds[r]), "lrcvt_mg_set_slab")
            nf = ctypes.c_int64()
            rc = _lib.check(L.lrcvt_mg_begin(eng.plan, S, site_pos.data_ptr(), site_comp.data_ptr(),
                                             eng.ss.data_ptr(), eng.dist.data_ptr(), ctypes.byref(nf), st),
                            "lrcvt_mg_begin")
            if rc > 0:
                raise ValueError(f"{rc} sites sit outside their recorded component")
            self._frontier.append(int(nf.value))
        self._run_rounds(1, stats)  # phase 1 (tessellation.py:151-156)
        self._frontier = []
        for r, eng in self.engines.items():
            nf = ctypes.c_int64()
            _lib.check(L.lrcvt_mg_phase2(eng.plan, S, site_comp.data_ptr(), ctypes.byref(nf), st), "phase2")
            self._frontier.append(int(nf.value))
        while True:  # phase 2 + verification sweeps (tessellation.py:170-189)
            self._run_rounds(2, stats)
            stats["sweeps"] += 1
            if self._round(2, 1, stats) == 0:
                break
        for r, eng in self.engines.items():
            a = ctypes.c_int64()
            _lib.check(L.lrcvt_mg_finish(eng.plan, eng.ss.data_ptr(), eng.state.data_ptr(), ctypes.byref(a), st),
                       "lrcvt_mg_finish")
            stats["assigned"] = int(a.value)
        return stats

    def any_engine(self) -> Engine:
        return next(iter(self.engines.values()))


def global_lrcvt(grid, labels, seeding, lloyd, coll=None):
    """lrcvt() (tessellation.py:251-275) in global mode: classification
    partitioned over the Collective's ranks, vote + move redundantly on each
    rank's replicated state. Returns (Tessellation, trace) on every rank."""
    from .seeding import Site, seed_sites, voxel_weights
    from .tessellation import Tessellation, lloyd_weight_mode, voxel_length

    torch = _lib.require_cuda()
    if labels.n_components == 0:
        raise ValueError("no connected components to tessellate")
    coll = coll or Emulated(1)
    sites, seed_report = seed_sites(grid, labels, seeding)
    weights = voxel_weights(grid, seeding)
    pos = np.array([s.position for s in sites], dtype=np.float64).reshape(-1, 3)
    sc = np.array([s.component_id for s in sites], dtype=np.int32)
    pos_d = torch.from_numpy(pos).cuda()
    sc_d = torch.from_numpy(sc).cuda()
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, max(len(sites), 1), coll)
    mode, w_d = lloyd_weight_mode(torch, grid, seeding, weights)
    vlen = voxel_length(grid.dims, grid.spacing)
    trace: list[float] = []
    for _ in range(lloyd.max_updates):
        gc.classify(pos_d, sc_d)
        new = None
        for eng in gc.engines.values():  # identical on every rank
            # the vote covers the whole (replicated) volume: full-range plan
            _lib.check(gc.L.lrcvt_mg_set_slab(eng.plan, 0, grid.dims[2]), "lrcvt_mg_set_slab")
            new, disp, _, _ = eng.centroidal(pos_d, sc_d, mode, w_d, 0.5 * vlen)
        pos_d = new
        d = disp.cpu().numpy()
        mean_ds = float(d.mean() / vlen) if d.size else 0.0
        trace.append(mean_ds)
        if mean_ds < lloyd.ds_tolerance:
            break
    st = gc.classify(pos_d, sc_d)
    eng = gc.any_engine()
    ss = eng.ss.cpu().numpy()
    final_pos = pos_d.cpu().numpy()
    final_sites = [Site((float(p[0]), float(p[1]), float(p[2])), int(c)) for p, c in zip(final_pos, sc)]
    has = np.zeros(max(labels.n_components, 1), dtype=bool)
    has[sc] = True
    report = {"rounds": st["rounds"], "sweeps": st["sweeps"],
              "components_without_sites": sorted(int(c.id) for c in labels.component_table if not has[c.id]),
              "assigned": st["assigned"], "seeding": seed_report, "updates": len(trace),
              "evaluations": st["evaluations"], "commits": st["commits"]}
    tess = Tessellation(grid.dims, grid.spacing, np.ascontiguousarray(ss[:, 0]), eng.dist.cpu().numpy(),
                        np.ascontiguousarray(ss[:, 1]), eng.state.cpu().numpy(),
                        np.ascontiguousarray(labels.component, dtype=np.int32), final_sites, report, weights)
    return tess, trace

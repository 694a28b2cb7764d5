"""Multi-GPU global mode: ONE tessellation over z-slabs of the whole volume,
bit-identical to the single-domain result (north star).

Design (csrc/mg.cuh): rank r OWNS planes [zlo_r, zhi_r).
Every rank keeps full-size per-voxel buffers, but only its own slab plus one
halo plane on each side is current locally:

  * evaluation: own frontier only (_eval_voxel, _kernels.py:147-246); the
    26-neighbourhood lies in slab + halo; the rare far reads -- the state of a
    shortcut node u = src(w) and the phi chains of the vote -- go to the
    owning rank's buffer through a peer pointer (NVLink P2P / CUDA IPC);
  * per round, only the improved proposals on the two boundary planes travel
    (to rank - 1 and rank + 1), and each rank commits its own proposals plus
    the received halo ones (_apply_and_enqueue, _kernels.py:285-334, with the
    enqueue restricted to the own slab); the global frontier size decides
    the next round (_run_phase, _kernels.py:337-385) and the sweeps
    (tessellation.py:170-189);
  * vote (_centroid_targets, _kernels.py:513-532) over the own slab: unit
    weights give exact integer partial sums, summed by an all-reduce; any
    other weights keep the reference's voxel-order fp64 chains -- each site's
    chain runs slab after slab, the running sums handed from rank to rank
    for the sites that straddle a slab boundary (all other sites in
    parallel); every rank then moves all sites from identical sums.

Every evaluation reads exactly the global pre-round state, so site_of / dist
/ src / state, rounds, sweeps and the E / C counters equal the single-domain
run. `Collective` hides where the ranks live:
  * `Emulated` -- all ranks in this process on one GPU; the ranks' steps run
    one after another on one stream (no kernel ever waits on another);
  * `TorchDist` -- one rank per process, torch.distributed (NCCL on GPUs,
    gloo with host staging in the CPU-coordinated tests); peer pointers via
    CUDA IPC handles exchanged at set-up.
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


def plane_inband(component: np.ndarray, dims) -> np.ndarray:
    """in-band voxels per z-plane"""
    nx, ny, nz = (int(d) for d in dims)
    return np.count_nonzero(np.asarray(component).reshape(nz, ny * nx) >= 0, axis=1).astype(np.float64)


def _cut(per: np.ndarray, world: int) -> list[tuple[int, int]]:
    """z-slabs of about equal total `per` (a cost per plane); every slab keeps at least one plane"""
    nz = per.size
    if world > nz:
        raise ValueError(f"cannot split {nz} planes into {world} non-empty slabs")
    cum = np.concatenate([[0.0], np.cumsum(per)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        z = int(np.searchsorted(cum, total * r / world, side="left"))
        z = min(max(z, cuts[-1] + 1), nz - (world - r))
        cuts.append(z)
    cuts.append(nz)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def balanced_slab_bounds(component: np.ndarray, dims, world: int) -> list[tuple[int, int]]:
    """z-slabs holding about equal numbers of in-band voxels (the work of a
    rank follows its in-band voxels, not its planes). Any bounds give the
    same results bit for bit."""
    return _cut(plane_inband(component, dims), world)


def cost_balanced_bounds(inband: np.ndarray, bounds, rank_cost) -> list[tuple[int, int]]:
    """Re-cut the slabs from measured per-rank costs: each plane's cost is its
    in-band voxel count times the measured cost per in-band voxel of the
    slab that holds it now; the new slabs carry equal predicted cost."""
    per = np.asarray(inband, dtype=np.float64).copy()
    for (lo, hi), c in zip(bounds, rank_cost):
        n = per[lo:hi].sum()
        per[lo:hi] *= (float(c) / n) if n > 0 else 0.0
    if per.sum() <= 0:
        return list(bounds)
    return _cut(per + 1e-12 * per.max(), len(bounds))


class _DevBuf:
    """A raw device allocation seen as a torch tensor (zero copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def as_tensor(torch, ptr, shape, typestr):
    return torch.as_tensor(_DevBuf(ptr, shape, typestr), device="cuda")


class Emulated:
    """All ranks live in this process (one GPU): collectives are host-side
    list operations over the ranks' tensors."""

    def __init__(self, world: int):
        self.world = world
        self.local_ranks = list(range(world))

    def sum_ints(self, per_rank: dict) -> list[int]:
        vals = list(per_rank.values())
        return [int(sum(v[i] for v in vals)) for i in range(len(vals[0]))]

    def exchange_halo(self, lo: dict, hi: dict, torch, extra: dict | None = None):
        """rank r receives hi of r - 1 and lo of r + 1 (uint8 tensors); with
        `extra` ({rank: [ints]}) also returns their sums over the ranks."""
        out = {}
        for r in self.local_ranks:
            parts = ([hi[r - 1]] if r > 0 else []) + ([lo[r + 1]] if r + 1 < self.world else [])
            parts = [p for p in parts if p.numel()]
            out[r] = torch.cat(parts) if parts else torch.empty(0, dtype=torch.uint8, device="cuda")
        if extra is None:
            return out
        return out, self.sum_ints(extra)

    def allreduce(self, per_rank: dict, op: str, torch):
        ts = list(per_rank.values())
        acc = ts[0].clone()
        for t in ts[1:]:
            if op == "sum":
                acc += t
            elif op == "min":
                torch.minimum(acc, t, out=acc)
            else:
                torch.maximum(acc, t, out=acc)
        return acc

    def chain(self, step, shape, torch):
        """carry = step(r, carry) for r = 0..world-1 in order; returns the last
        rank's carry (the final running sums), identical on every rank."""
        carry = None
        for r in range(self.world):
            carry = step(r, carry)
        return carry

    def gather_floats(self, per_rank: dict) -> list[float]:
        return [float(per_rank[r]) for r in range(self.world)]

    def peer_pointers(self, own: dict):
        """own: {rank: (ss_ptr, dist_ptr)} -> lists over all ranks."""
        return [own[r][0] for r in range(self.world)], [own[r][1] for r in range(self.world)]


class TorchDist:
    """One rank per process over torch.distributed: NCCL on CUDA tensors for
    the GPU path; device="cpu" stages every collective through host memory
    (gloo) -- the CPU-coordinated tests of the protocol."""

    def __init__(self, group=None, device: str | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if device is None:  # NCCL moves CUDA tensors; gloo (and any other backend) stages through host memory
            device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        self.device = device
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local_ranks = [self.rank]
        self._opened = []
        import torch

        self.home = "cuda" if torch.cuda.is_available() else "cpu"  # where results are handed back

    def _to(self, t):
        return t.to(self.device) if str(t.device) != self.device else t

    def all_counts(self, local: list[int]) -> list[int]:
        import torch

        t = torch.tensor(local, dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(v) for x in out for v in x.tolist()]

    def gather_floats(self, per_rank: dict) -> list[float]:
        import torch

        t = torch.tensor([float(per_rank[self.rank])], dtype=torch.float64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [float(x.item()) for x in out]

    def sum_ints(self, per_rank: dict) -> list[int]:
        import torch

        t = torch.tensor(per_rank[self.rank], dtype=torch.int64, device=self.device)
        self.dist.all_reduce(t, group=self.group)
        return [int(v) for v in t.tolist()]

    def _all_bytes(self, local, torch):
        """all ranks' uint8 tensors (variable sizes) in rank order."""
        n = self.all_counts([int(local.numel())])
        m = max(n)
        if m == 0:
            return [local[:0]] * self.world
        pad = torch.zeros(m, dtype=torch.uint8, device=self.device)
        pad[: local.numel()] = self._to(local)
        out = [torch.empty(m, dtype=torch.uint8, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(out, pad, group=self.group)
        return [o[:c] for o, c in zip(out, n)]

    def all_props(self, local: list, torch):
        """Concatenate every rank's proposal bytes in rank order."""
        return torch.cat(self._all_bytes(local[0], torch))

    def exchange_halo(self, lo: dict, hi: dict, torch, extra: dict | None = None):
        """rank r sends lo to r - 1 and hi to r + 1 and receives hi of r - 1 and
        lo of r + 1: one all-gather of the list sizes (and of `extra`, whose
        sums over the ranks come back too), then point-to-point transfers
        between neighbours only (NVLink P2P under NCCL)."""
        r, world = self.rank, self.world
        mine_lo, mine_hi = lo[r], hi[r]
        ex = list(extra[r]) if extra is not None else []
        k = 2 + len(ex)
        g = self.all_counts([int(mine_lo.numel()), int(mine_hi.numel())] + ex)
        n = [g[q * k + j] for q in range(world) for j in range(2)]
        sums = [sum(g[q * k + 2 + j] for q in range(world)) for j in range(len(ex))]
        P2POp = self.dist.P2POp
        ops, got = [], []
        if r > 0 and n[2 * (r - 1) + 1]:  # hi of r - 1
            buf = torch.empty(n[2 * (r - 1) + 1], dtype=torch.uint8, device=self.device)
            ops.append(P2POp(self.dist.irecv, buf, r - 1, self.group))
            got.append(buf)
        if r + 1 < world and n[2 * (r + 1)]:  # lo of r + 1
            buf = torch.empty(n[2 * (r + 1)], dtype=torch.uint8, device=self.device)
            ops.append(P2POp(self.dist.irecv, buf, r + 1, self.group))
            got.append(buf)
        if r > 0 and mine_lo.numel():
            ops.append(P2POp(self.dist.isend, self._to(mine_lo), r - 1, self.group))
        if r + 1 < world and mine_hi.numel():
            ops.append(P2POp(self.dist.isend, self._to(mine_hi), r + 1, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        out = torch.cat(got) if got else torch.empty(0, dtype=torch.uint8, device=self.device)
        if extra is None:
            return {r: out.to(self.home)}
        return {r: out.to(self.home)}, sums

    def allreduce(self, per_rank: dict, op: str, torch):
        t = self._to(per_rank[self.rank].clone())
        red = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX}[op]
        self.dist.all_reduce(t, op=red, group=self.group)
        return t.to(self.home)

    def chain(self, step, shape, torch):
        r = self.rank
        carry = None
        if r > 0:
            buf = torch.empty(shape, dtype=torch.float64, device=self.device)
            self.dist.recv(buf, src=r - 1, group=self.group)
            carry = buf.to(self.home)
        carry = step(r, carry)
        if r + 1 < self.world:
            if self.home == "cuda":
                torch.cuda.current_stream().synchronize()
            self.dist.send(self._to(carry), dst=r + 1, group=self.group)
        final = self._to(carry) if r == self.world - 1 else torch.empty(shape, dtype=torch.float64,
                                                                      device=self.device)
        self.dist.broadcast(final, src=self.world - 1, group=self.group)
        return final.to(self.home)

    def peer_pointers(self, own: dict):
        """CUDA IPC: export this rank's state buffers, open every other rank's."""
        import torch

        L = _lib.lib()
        h = (ctypes.c_uint8 * 128)()
        base = ctypes.addressof(h)
        ss, dist = own[self.rank]
        _lib.check(L.lrcvt_ipc_export(ss, base), "ipc export")
        _lib.check(L.lrcvt_ipc_export(dist, base + 64), "ipc export")
        mine = torch.tensor(list(bytes(h)), dtype=torch.uint8, device=self.device)
        allh = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(allh, mine, group=self.group)
        pss, pdist = [], []
        for q, t in enumerate(allh):
            if q == self.rank:
                pss.append(ss)
                pdist.append(dist)
                continue
            raw = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
            a, b = ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(L.lrcvt_ipc_open(ctypes.addressof(raw), ctypes.byref(a)), "ipc open")
            _lib.check(L.lrcvt_ipc_open(ctypes.addressof(raw) + 64, ctypes.byref(b)), "ipc open")
            self._opened += [a.value, b.value]
            pss.append(a.value)
            pdist.append(b.value)
        return pss, pdist

    def close(self):
        L = _lib.lib()
        for p in self._opened:
            L.lrcvt_ipc_close(p)
        self._opened = []


class GlobalClassifier:
    """Slab-partitioned voronoi_classify and centroidal update over a
    Collective. Each local rank owns an Engine (plan with slab bounds and
    peer view); its plan-owned state buffers are current on the own slab
    (engine.ss / engine.dist views of them, engine.state its state bits)."""

    def __init__(self, dims, spacing, component: np.ndarray, n_components: int, max_sites: int, coll,
                 bounds=None):
        torch = self.torch = _lib.require_cuda()
        self.L = _lib.lib()
        self.coll = coll
        self.dims = tuple(int(d) for d in dims)
        self.spacing = tuple(float(s) for s in spacing)
        self.n = int(np.prod(self.dims))
        # z-slabs with about equal in-band voxel counts unless given ([(zlo, zhi)] per rank)
        self._inband = plane_inband(component, self.dims)
        self.bounds = list(bounds) if bounds is not None else _cut(self._inband, coll.world)
        self.engines = {}
        comp_dev = None
        own = {}
        for r in coll.local_ranks:
            eng = Engine(self.dims, spacing, component, n_components, max_sites, comp_dev, alloc_state=False)
            comp_dev = eng.comp  # replicated labels shared between in-process ranks
            lo, hi = self.bounds[r]
            _lib.check(self.L.lrcvt_mg_set_slab(eng.plan, lo, hi), "lrcvt_mg_set_slab")
            a, b = ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(self.L.lrcvt_mg_state(eng.plan, ctypes.byref(a), ctypes.byref(b)), "lrcvt_mg_state")
            eng.ss = as_tensor(torch, a.value, (self.n, 2), "<i4")
            eng.dist = as_tensor(torch, b.value, (self.n,), "<f8")
            own[r] = (a.value, b.value)
            self.engines[r] = eng
        self.timing = False  # per-rank device time (CUDA events around every rank's calls)
        self._ev = {r: [] for r in self.engines}
        self._lib_ms = {r: {} for r in self.engines}
        self.calls = {r: {} for r in self.engines}  # timed calls per category (timing mode)
        self._peers = coll.peer_pointers(own)
        self._set_peers()
        self._S = 0

    def _set_peers(self):
        world = self.coll.world
        pss, pdist = self._peers
        zb = (ctypes.c_int64 * (world + 1))(*([lo for lo, _ in self.bounds] + [self.dims[2]]))
        arr_ss = (ctypes.c_void_p * world)(*pss)
        arr_d = (ctypes.c_void_p * world)(*pdist)
        for r, eng in self.engines.items():
            _lib.check(self.L.lrcvt_mg_set_peers(eng.plan, world, zb, arr_ss, arr_d), "lrcvt_mg_set_peers")

    def rebalance(self, rank_cost: dict) -> list[tuple[int, int]]:
        """Move the slab bounds so that every rank carries the same predicted
        cost, from the costs measured on the current bounds ({local rank:
        cost}; gathered over the collective). Results stay bit-identical:
        the bounds only decide who computes what. Returns the new bounds."""
        costs = self.coll.gather_floats(rank_cost)
        new = cost_balanced_bounds(self._inband, self.bounds, costs)
        if new != self.bounds:
            self.bounds = new
            for r, eng in self.engines.items():
                lo, hi = new[r]
                _lib.check(self.L.lrcvt_mg_set_slab(eng.plan, lo, hi), "lrcvt_mg_set_slab")
            self._set_peers()
        return new

    def reuse_sites(self, on: bool):
        """keep each rank's eligible list across classifies (a Lloyd loop: the
        site components do not change between iterations)"""
        for eng in self.engines.values():
            _lib.check(self.L.lrcvt_plan_reuse_eligible(eng.plan, 2 if on else 0), "reuse_eligible")

    def _st(self):
        return _lib.stream_handle(self.torch)

    def set_timing(self, on: bool):
        """per-rank device time: CUDA events around each rank's non-synchronising calls here, and the
        library's own events around the kernels of its synchronising steps (lrcvt_mg_timing: a host
        round trip inside a step is not device work)"""
        self.timing = on
        for eng in self.engines.values():
            _lib.check(self.L.lrcvt_mg_timing(eng.plan, 1 if on else 0, None), "lrcvt_mg_timing")

    def _t(self, r, fn, synced=False, cat="other"):
        """run fn() for rank r, bracketed by CUDA events when timing (synced
        steps are timed by the library); the time is booked under cat"""
        if not self.timing:
            return fn()
        if synced:
            out = fn()
            ms = ctypes.c_double()
            _lib.check(self.L.lrcvt_mg_timing(self.engines[r].plan, 1, ctypes.byref(ms)), "mg timing")
            if callable(cat):
                cat = cat()
            self._lib_ms[r][cat] = self._lib_ms[r].get(cat, 0.0) + ms.value
            self.calls[r][cat] = self.calls[r].get(cat, 0) + 1
            return out
        torch = self.torch
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        self._ev[r].append((cat, a, b))
        return out

    def rank_ms(self, breakdown: bool = False) -> dict:
        """device milliseconds spent in each local rank's own kernels since the
        last call (emulated ranks share one GPU and never overlap); with
        breakdown, {rank: {step category: ms}}"""
        self.torch.cuda.synchronize()
        cats = {r: dict(self._lib_ms[r]) for r in self.engines}
        for r, evs in self._ev.items():
            for cat, a, b in evs:
                cats[r][cat] = cats[r].get(cat, 0.0) + a.elapsed_time(b)
        self._ev = {r: [] for r in self.engines}
        self._lib_ms = {r: {} for r in self.engines}
        for r, eng in self.engines.items():
            ms = ctypes.c_double()
            _lib.check(self.L.lrcvt_mg_timing(eng.plan, 1 if self.timing else 0, ctypes.byref(ms)), "mg timing")
            cats[r]["other"] = cats[r].get("other", 0.0) + ms.value
        return cats if breakdown else {r: sum(c.values()) for r, c in cats.items()}

    def _eval_all(self, phase: int, sweep: int):
        """eval on every local rank: ({rank: evaluated}, lo lists, hi lists)"""
        L, st = self.L, self._st()
        counts, lo, hi = {}, {}, {}
        for r, eng in self.engines.items():
            ne, nlo, nhi = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            self._t(r, lambda: _lib.check(L.lrcvt_mg_eval(eng.plan, phase, sweep, ctypes.byref(ne), ctypes.byref(nlo),
                                                          ctypes.byref(nhi), st), "lrcvt_mg_eval"), synced=True,
                    cat=lambda: f"eval_p{phase}_" + _size_class(ne.value))
            counts[r] = int(ne.value)
            lo[r] = self._bytes(L.lrcvt_mg_boundary(eng.plan, 0), int(nlo.value))
            hi[r] = self._bytes(L.lrcvt_mg_boundary(eng.plan, 1), int(nhi.value))
        return counts, lo, hi

    def _commit_all(self, halo: dict, sweep: int) -> dict:
        """commit on every local rank: {rank: (own next frontier, own proposals committed)}"""
        L, st = self.L, self._st()
        done = {}
        for r, eng in self.engines.items():
            h = halo[r]
            nn, nc = ctypes.c_int64(), ctypes.c_int64()
            self._t(r, lambda: _lib.check(L.lrcvt_mg_commit(eng.plan, h.data_ptr() if h.numel() else None,
                                                            h.numel() // PROP_BYTES, sweep, ctypes.byref(nn),
                                                            ctypes.byref(nc), st),
                                          "lrcvt_mg_commit"), synced=True, cat="commit")
            done[r] = (int(nn.value), int(nc.value))
        return done

    def _run_rounds(self, phase: int, stats: dict):
        """Relaxation rounds until the global frontier is empty. One
        collective per round besides the halo transfers: the all-gather of
        the boundary-list sizes also carries every rank's frontier size and
        its commits of the previous round, so the loop ends on a round whose
        every frontier was empty (an eval of nothing) instead of a separate
        all-reduce after each commit."""
        if self._frontier <= 0:
            return
        prev = {r: 0 for r in self.engines}
        while True:
            counts, lo, hi = self._eval_all(phase, 0)
            halo, tot = self.coll.exchange_halo(lo, hi, self.torch, {r: [counts[r], prev[r]] for r in self.engines})
            stats["commits"] += tot[1]
            if tot[0] == 0:
                break
            stats["rounds"] += 1
            stats["evaluations"] += tot[0]
            prev = {r: nc for r, (_, nc) in self._commit_all(halo, 0).items()}
        self._frontier = 0

    def _sweep(self, stats: dict) -> int:
        """a verification sweep (phase 2) on all ranks; returns the global
        number of improved proposals and sets the global frontier size"""
        counts, lo, hi = self._eval_all(2, 1)
        halo = self.coll.exchange_halo(lo, hi, self.torch)
        done = self._commit_all(halo, 1)
        tot = self.coll.sum_ints({r: [done[r][0], counts[r], done[r][1]] for r in self.engines})
        self._frontier = tot[0]
        stats["evaluations"] += tot[1]
        stats["commits"] += tot[2]
        return tot[2]

    def _bytes(self, ptr, n):
        torch = self.torch
        if n == 0 or not ptr:
            return torch.empty(0, dtype=torch.uint8, device="cuda")
        return as_tensor(torch, ptr, (n * PROP_BYTES,), "|u1").clone()

    def classify(self, site_pos, site_comp) -> dict:
        """site_pos float64[S,3], site_comp int32[S] on the device; returns
        the report counters (rounds, sweeps, assigned, evaluations, commits)."""
        L, st = self.L, self._st()
        S = int(site_pos.shape[0])
        self._S = S
        stats = {"rounds": 0, "sweeps": 0, "evaluations": 0, "commits": 0}
        front, bad = {}, 0
        for r, eng in self.engines.items():
            if S > eng.max_sites:
                raise ValueError("more sites than the global classifier was sized for")
            nf = ctypes.c_int64()
            rc = self._t(r, lambda: _lib.check(L.lrcvt_mg_begin(eng.plan, S, site_pos.data_ptr(),
                                                                site_comp.data_ptr(), eng.ss.data_ptr(),
                                                                eng.dist.data_ptr(), ctypes.byref(nf), st),
                                               "lrcvt_mg_begin"), synced=True, cat="begin")
            bad = max(bad, rc)
            front[r] = [int(nf.value)]
        if bad > 0:
            raise ValueError(f"{bad} sites sit outside their recorded component")
        self._frontier = self.coll.sum_ints(front)[0]
        self._run_rounds(1, stats)  # phase 1 (tessellation.py:151-156)
        front = {}
        for r, eng in self.engines.items():
            nf = ctypes.c_int64()
            self._t(r, lambda: _lib.check(L.lrcvt_mg_phase2(eng.plan, S, site_comp.data_ptr(), ctypes.byref(nf),
                                                            st), "phase2"), synced=True, cat="phase2")
            front[r] = [int(nf.value)]
        self._frontier = self.coll.sum_ints(front)[0]
        while True:  # phase 2 + verification sweeps (tessellation.py:170-189)
            self._run_rounds(2, stats)
            stats["sweeps"] += 1
            if self._sweep(stats) == 0:
                break
        assigned = {}
        for r, eng in self.engines.items():
            a = ctypes.c_int64()
            self._t(r, lambda: _lib.check(L.lrcvt_mg_finish(eng.plan, eng.ss.data_ptr(), eng.state.data_ptr(),
                                                            ctypes.byref(a), st), "lrcvt_mg_finish"), synced=True,
                    cat="finish")
            assigned[r] = [int(a.value)]
        stats["assigned"] = self.coll.sum_ints(assigned)[0]
        return stats

    def centroidal(self, site_pos, site_comp, weight_mode: int, weights, backoff: float):
        """centroidal_update (tessellation.py:211-248) over the slabs; returns
        (new_pos, disp, empty) -- identical on every rank."""
        torch, L, st = self.torch, self.L, self._st()
        S = int(site_pos.shape[0])
        sx, sy, sz = self.spacing
        exact = (weight_mode == _lib.W_ONES and all(_pow2(s) for s in self.spacing)
                 and max(self.dims) <= (1 << 20))
        if exact:
            acc = {}
            for r, eng in self.engines.items():
                a = torch.empty((4, S), dtype=torch.int64, device="cuda")
                self._t(r, lambda: _lib.check(L.lrcvt_mg_vote_exact(eng.plan, S, eng.ss.data_ptr(), a.data_ptr(), st),
                                              "vote"), synced=True, cat="vote")
                acc[r] = a
            red = self.coll.allreduce(acc, "sum", torch)
            sums = torch.empty((4, S), dtype=torch.float64, device="cuda")
            eng0 = next(iter(self.engines.values()))
            _lib.check(L.lrcvt_mg_vote_exact_finish(eng0.plan, S, red.data_ptr(), sums.data_ptr(), st), "finish")
        else:
            boxes, res = {}, {}
            for r, eng in self.engines.items():
                b = torch.empty((6, S), dtype=torch.int32, device="cuda")
                self._t(r, lambda: _lib.check(L.lrcvt_mg_vote_box(eng.plan, S, eng.ss.data_ptr(), b.data_ptr(), st),
                                              "vote box"), synced=True, cat="vote_box")
                boxes[r] = b
            lo = self.coll.allreduce({r: b[:3].contiguous() for r, b in boxes.items()}, "min", torch)
            hi = self.coll.allreduce({r: b[3:].contiguous() for r, b in boxes.items()}, "max", torch)
            box = torch.cat([lo, hi]).contiguous()
            wp = _lib.ptr(weights)
            for r, eng in self.engines.items():  # sites whose box starts in the own slab: all ranks at once
                out = torch.zeros((4, S), dtype=torch.float64, device="cuda")
                self._t(r, lambda: _lib.check(L.lrcvt_mg_vote_scan(eng.plan, S, site_comp.data_ptr(), weight_mode, wp,
                                                                   1, box.data_ptr(), None, out.data_ptr(), st),
                                              "vote scan"), synced=True, cat="vote_scan1")
                res[r] = out

            def step(r, carry):  # sites continuing from earlier slabs, then the hand-over
                eng = self.engines[r]
                if carry is not None:
                    self._t(r, lambda: _lib.check(L.lrcvt_mg_vote_scan(eng.plan, S, site_comp.data_ptr(), weight_mode,
                                                                       wp, 2, box.data_ptr(), carry.data_ptr(),
                                                                       res[r].data_ptr(), st), "vote scan"), synced=True, cat="vote_scan2")
                out = torch.empty((4, S), dtype=torch.float64, device="cuda")
                self._t(r, lambda: _lib.check(L.lrcvt_mg_vote_carry(eng.plan, S, box.data_ptr(), res[r].data_ptr(),
                                                                    carry.data_ptr() if carry is not None else None,
                                                                    out.data_ptr(), st), "vote carry"), synced=True, cat="vote_carry")
                return out

            sums = self.coll.chain(step, (4, S), torch)
        new_pos = disp = None
        empty = ctypes.c_int64()
        for r, eng in self.engines.items():  # every rank moves every site (identical inputs)
            new_pos = torch.empty((S, 3), dtype=torch.float64, device="cuda")
            disp = torch.empty(S, dtype=torch.float64, device="cuda")
            np_, dp_ = new_pos, disp
            self._t(r, lambda: _lib.check(L.lrcvt_mg_move(eng.plan, S, site_pos.data_ptr(), site_comp.data_ptr(),
                                                          sums.data_ptr(), float(backoff), np_.data_ptr(),
                                                          dp_.data_ptr(), ctypes.byref(empty), st), "lrcvt_mg_move"), synced=True,
                          cat="move")
        return new_pos, disp, int(empty.value)

    def own_slab(self, r):
        """(voxel range, engine) of rank r's own slab."""
        lo, hi = self.bounds[r]
        nxy = self.dims[0] * self.dims[1]
        return lo * nxy, hi * nxy, self.engines[r]

    def any_engine(self) -> Engine:
        return next(iter(self.engines.values()))


def _size_class(n: int) -> str:
    """timing category of a round by its per-rank frontier size"""
    return "small" if n <= 2048 else ("mid" if n <= 65536 else "big")


def _pow2(s: float) -> bool:
    m, _ = math.frexp(s)
    return s > 0 and m == 0.5


def global_lrcvt(grid, labels, seeding, lloyd, coll=None):
    """lrcvt() (tessellation.py:251-275) in global mode: classification and
    vote partitioned over the Collective's ranks. Returns (Tessellation,
    trace); the per-voxel arrays are assembled from the local ranks' slabs
    (every slab when all ranks are local)."""
    from .seeding import seed_sites, voxel_weights
    from .tessellation import Tessellation, lloyd_weight_mode, make_sites, voxel_length

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
    gc.reuse_sites(True)  # site components fixed for the whole loop
    try:
        for _ in range(lloyd.max_updates):
            gc.classify(pos_d, sc_d)
            pos_d, disp, _ = gc.centroidal(pos_d, sc_d, mode, w_d, 0.5 * vlen)
            d = disp.cpu().numpy()
            mean_ds = float(d.mean() / vlen) if d.size else 0.0
            trace.append(mean_ds)
            if mean_ds < lloyd.ds_tolerance:
                break
        st = gc.classify(pos_d, sc_d)
    finally:
        gc.reuse_sites(False)
    n = grid.size
    site_of = np.full(n, -1, np.int32)
    src = np.full(n, -1, np.int32)
    dist = np.full(n, np.inf)
    state = np.zeros(n, np.uint8)
    for r in gc.engines:
        v0, v1, eng = gc.own_slab(r)
        ss = eng.ss[v0:v1].cpu().numpy()
        site_of[v0:v1] = ss[:, 0]
        src[v0:v1] = ss[:, 1]
        dist[v0:v1] = eng.dist[v0:v1].cpu().numpy()
        state[v0:v1] = eng.state[v0:v1].cpu().numpy()
    final_pos = pos_d.cpu().numpy()
    final_sites = make_sites(final_pos, sc)
    has = np.zeros(max(labels.n_components, 1), dtype=bool)
    has[sc] = True
    report = {"rounds": st["rounds"], "sweeps": st["sweeps"],
              "components_without_sites": sorted(int(c.id) for c in labels.component_table if not has[c.id]),
              "assigned": st["assigned"], "seeding": seed_report, "updates": len(trace),
              "evaluations": st["evaluations"], "commits": st["commits"]}
    tess = Tessellation(grid.dims, grid.spacing, site_of, dist, src, state,
                        np.ascontiguousarray(labels.component, dtype=np.int32), final_sites, report, weights)
    return tess, trace

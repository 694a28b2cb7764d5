"""Benchmark: CVT-iteration voxels/s of the geodesic LSRCVT hot path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

A step is one Lloyd iteration (voronoi_classify + centroidal_update: LOS
classification, phi-propagated vote, clamped site move) over the whole volume;
value = voxels x steps / device time. The default workload
is C4 (BASELINE.json configs[3], the largest configuration quoted for ONE
GPU: 512^3 random-smooth, 3 bands, 32 776 'g'-weighted sites); c1-c3 and c5
(1024^3 on one B200) are selectable with --config.

--gpus N > 1 outside torchrun re-launches this script under
torch.distributed.run (one rank per GPU, 127.0.0.1). --mode global (the
default for N > 1) splits ONE volume into z-slabs (strong scaling); --mode
blocks runs one independent volume per rank (weak scaling).

--impl reference times the reference algorithm's CPU implementation (the C
oracle port in oracle/, all host threads) on the same config: one Lloyd
iteration per step, timed until K steps or --ref-budget seconds (a bounded
sample); rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(kind="spiral", dims=(256, 256, 1), iso=[0.3, 0.55, 0.8],
               seeding=dict(alpha=64, gamma=1.0, weight_field="g", block_size=16, seed=0),
               label="C1 2D 256^2 spiral, 2 nested bands, 69 g-weighted sites"),
    "c2": dict(kind="gaussian-mix", dims=(128, 128, 128), iso=[0.3, 0.7],
               seeding=dict(alpha=512, weight_field="g", seed=0),
               label="C2 3D 128^3 gaussian-mix, 1 band, 512 g-weighted sites"),
    "c3": dict(kind="horseshoe", dims=(256, 256, 256), iso=[0.0, 0.12, 0.3],
               seeding=dict(alpha=4096, seed=0),
               label="C3 3D 256^3 horseshoe shells, 2 bands, 4097 unweighted sites"),
    "c4": dict(kind="random-smooth", dims=(512, 512, 512), iso=[0.35, 0.5, 0.65, 0.8],
               seeding=dict(alpha=32768, weight_field="g", seed=0),
               label="C4 3D 512^3 random-smooth, 3 bands, 32k g-weighted sites"),
    # north-star volume on ONE B200; fields generated on the GPU (synth_c5)
    "c5": dict(kind="c5-helix", dims=(1024, 1024, 1024), iso=[0.55, 0.75, 0.95],
               seeding=dict(alpha=262144, weight_field="g", seed=0),
               label="C5 3D 1024^3 helical two-field, 2 bands, 256k g-weighted sites"),
}
L2_BYTES = 126 * 2**20


def bench_config(cfg, n, S, inband):
    """The `config` object of the JSON line -- identical in both arms."""
    state_bytes = n * (8 + 8 + 4 + 1)
    l2 = ("flushed between steps (256 MiB write)" if state_bytes < 2 * L2_BYTES
          else f"inputs larger than L2 (per-voxel state {state_bytes / 2**20:.0f} MiB > 126 MiB)")
    return {"workload": cfg["label"], "dims": list(cfg["dims"]), "voxels": int(n), "sites": int(S),
            "inband": int(inband), "step": "one Lloyd iteration (voronoi_classify + centroidal_update)",
            "l2": l2}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def synth_c5(dims, seed):
    """C5 input: f = the 3D helical spiral formula of
    synth_field (grid.py:268-275) and g = smooth value noise (a 17^3 lattice of
    uniform randoms, trilinear), both computed on the GPU in float64 and stored
    as float32 -- the numpy generator would need ~100 GB of host temporaries
    at 1024^3. Synthetic input generation only; not part of any timed region."""
    import torch

    from paper_2208_06970_b200.grid import VoxelGrid

    nx, ny, nz = dims
    dev = "cuda"
    f = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)
    xs = torch.arange(nx, dtype=torch.float64, device=dev) + 0.5
    ys = torch.arange(ny, dtype=torch.float64, device=dev) + 0.5
    yy, xx = torch.meshgrid(ys - ny / 2, xs - nx / 2, indexing="ij")
    theta = torch.atan2(yy, xx)
    r = torch.sqrt(xx * xx + yy * yy)
    base = 2.0 * theta + (10.0 / max(nx, ny)) * 2 * np.pi * r / 4.0
    amp = torch.clamp(r / (0.55 * min(nx, ny)), 0, 1.2)
    for z in range(nz):
        f[z] = (0.5 * (1.0 + torch.cos(base + 2 * np.pi * (z + 0.5) / nz)) * amp).to(torch.float32)
    del xs, ys, yy, xx, theta, r, base, amp
    lat = torch.from_numpy(np.random.default_rng(seed + 1).random((1, 1, 17, 17, 17))).to(dev)
    g = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)
    step = 64
    for z0 in range(0, nz, step):
        zc = min(step, nz - z0)
        # trilinear value noise on a lattice with one node every nx/16 voxels
        zz = (torch.arange(z0, z0 + zc, dtype=torch.float64, device=dev) + 0.5) * 16.0 / nz
        yv = (torch.arange(ny, dtype=torch.float64, device=dev) + 0.5) * 16.0 / ny
        xv = (torch.arange(nx, dtype=torch.float64, device=dev) + 0.5) * 16.0 / nx
        grid = torch.stack(torch.meshgrid(zz, yv, xv, indexing="ij")[::-1], dim=-1) / 8.0 - 1.0
        g[z0:z0 + zc] = torch.nn.functional.grid_sample(lat, grid[None], mode="bilinear",
                                                         align_corners=True)[0, 0].to(torch.float32)
        del grid
    out = VoxelGrid(dims=tuple(dims), spacing=(1.0, 1.0, 1.0),
                    fields={"f": f.reshape(-1).cpu().numpy(), "g": g.reshape(-1).cpu().numpy()})
    del f, g
    torch.cuda.empty_cache()
    return out


def build_workload(cfg, rank, use_gpu_masks=True):
    from paper_2208_06970_b200 import (IsobandSpec, SeedingParams, classify_isobands, label_components,
                                       seed_sites, synth_field, voxel_weights)

    grid = synth_c5(cfg["dims"], rank) if cfg["kind"] == "c5-helix" else synth_field(cfg["kind"], cfg["dims"], rank)
    spec = IsobandSpec("f", cfg["iso"])
    if use_gpu_masks:
        labels = label_components(classify_isobands(grid, spec))
    else:
        from oracle import oracle
        from paper_2208_06970_b200.grid import ComponentInfo, LabelMap

        layer = oracle.isobands(grid.fields["f"], spec.iso_values)
        comp, table = oracle.label_components(layer, grid.dims, spec.n_bands)
        labels = LabelMap(grid.dims, layer, comp,
                          [ComponentInfo(t["id"], t["layer"], t["voxel_count"], tuple(t["bbox"]), (0, 0))
                           for t in table], spec.iso_values, "f")
    params = SeedingParams(**cfg["seeding"])
    sites, _ = seed_sites(grid, labels, params, device=use_gpu_masks)
    weights = voxel_weights(grid, params) if grid.size <= (1 << 28) else None  # host f64 copy: e2e / CPU arm only
    return grid, labels, params, sites, weights


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args, cfg, world, rank):
    """CPU arm: the oracle port of the reference algorithm (oracle/lrcvt_oracle.c:
    the numba kernels restated in C, OpenMP eval + serial commit like the
    reference), all host threads, on the same workload. One step = one full
    Lloyd iteration from the previous step's sites; warm-up is one iteration
    (a CPU port has no JIT or allocator warm-up beyond the first touch), then
    steps are timed until K are done or --ref-budget seconds have elapsed."""
    if rank != 0:
        return
    from oracle import oracle

    oracle.build()
    oracle.set_num_threads(os.cpu_count() or 1)  # all host threads, whatever OMP_NUM_THREADS says
    grid, labels, params, sites, weights = build_workload(cfg, 0, use_gpu_masks=False)
    n = grid.size
    pos = np.array([s.position for s in sites])
    sc = np.array([s.component_id for s in sites], np.int32)
    w = None if params.weight_field is None else weights
    comp = labels.component
    inband = int(np.count_nonzero(comp >= 0))

    def step(p):
        c = oracle.classify(grid.dims, grid.spacing, comp, p, sc, labels.n_components)
        return oracle.centroidal(grid.dims, grid.spacing, comp, c["site_of"], c["src"], w, p, sc)["new_pos"]

    warm = min(args.warmup, 1)
    for _ in range(warm):
        pos = step(pos)
    t0 = time.perf_counter()
    done = 0
    while done < args.steps:
        pos = step(pos)
        done += 1
        el = time.perf_counter() - t0
        if el + el / done > args.ref_budget:  # the next step would overrun the budget
            break
    dt = time.perf_counter() - t0
    value = n * done / dt
    threads = oracle.num_threads()
    sample = (f"{done} full Lloyd iteration(s) of the workload after {warm} warm-up iteration(s), timed "
              f"{'(all ' + str(args.steps) + ' steps)' if done == args.steps else f'(budget {args.ref_budget:.0f} s reached)'}")
    line = {
        "impl": "reference", "metric": "CVT-iteration voxels/s", "value": value, "unit": "voxels/s",
        "n_gpus": world, "steps": args.steps, "steps_timed": done, "warmup": args.warmup, "warmup_timed": warm,
        "ms_per_step": 1e3 * dt / done, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(cfg, n, len(sites), inband),
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def seeding_pass(grid, labels, params):
    """Seeding stage: the GPU mass table alone and the
    whole seed_sites (GPU table + host numpy draw), wall clock; the host numpy
    table beside it on volumes where it takes seconds, not minutes."""
    import torch

    from paper_2208_06970_b200.seeding import component_masses, component_masses_device, seed_sites

    def wall(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return 1e3 * (time.perf_counter() - t0)

    component_masses_device(grid, labels, params)  # warm-up (allocator, CUB)
    out = {"masses_gpu_ms": wall(lambda: component_masses_device(grid, labels, params)),
           "seed_sites_ms": wall(lambda: seed_sites(grid, labels, params, device=True))}
    if grid.size <= (1 << 22):
        out["masses_host_numpy_ms"] = wall(lambda: component_masses(grid, labels, params))
    out["note"] = "wall clock incl. D2H of the grouped voxel/weight lists; the draw (Generator.choice) is host numpy"
    return out


def layout_pass(grid, labels, eng, S):
    """Layout record pass: the device select + sort +
    pack of the record block (CUDA events, device-resident inputs) and the
    whole build_and_write to a scratch file (wall clock, D2H + disk)."""
    import ctypes
    import tempfile

    import torch

    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.layout import record_dtype

    L = _lib.lib()
    names = grid.field_names()
    nx, ny, nz = grid.dims
    fields = [torch.from_numpy(grid.fields[k]).cuda() for k in names]
    ptrs = (ctypes.c_void_p * len(fields))(*[t.data_ptr() for t in fields])
    site_of = eng.ss[:, 0].contiguous()
    r_cap = eng.inband
    dt = record_dtype(len(names))
    rec = torch.empty(r_cap * dt.itemsize, dtype=torch.uint8, device="cuda")
    key = torch.empty(r_cap, dtype=torch.int32, device="cuda")
    nc = max(labels.n_components, 1)
    first = torch.empty(nc, dtype=torch.int64, device="cuda")
    count = torch.empty(nc, dtype=torch.int64, device="cuda")
    got = ctypes.c_int64()
    st = _lib.stream_handle(torch)

    def run():
        _lib.check(L.lrcvt_layout_records(nx, ny, nz, len(names), ptrs, eng.comp.data_ptr(), site_of.data_ptr(),
                                          labels.n_components, S, r_cap, rec.data_ptr(), key.data_ptr(),
                                          first.data_ptr(), count.data_ptr(), ctypes.byref(got), st), "layout")

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    r = int(got.value)
    bytes_moved = r * (4 + 4 + 8 + dt.itemsize) + 4 * len(names) * r + 4 * grid.size
    return {"records": r, "record_bytes": r * dt.itemsize, "device_ms": ms,
            "voxels_per_s": grid.size / (ms / 1e3), "algorithmic_GBps": bytes_moved / (ms / 1e3) / 1e9,
            "note": "lrcvt_layout_records: in-band select, (component, region, voxel) radix sort, record pack; "
                    "bytes = component scan 4N + per record key/voxel/region 16 B + gathers 4m + record out"}


def adjacency_pass(grid, eng, S):
    """Site adjacency face scan, CUDA events."""
    import ctypes

    import torch

    from paper_2208_06970_b200 import _lib

    L = _lib.lib()
    nx, ny, nz = grid.dims
    site_of = eng.ss[:, 0].contiguous()
    cap = 32 * S + 1024
    edges = torch.empty((cap, 2), dtype=torch.int64, device="cuda")
    got = ctypes.c_int64()
    st = _lib.stream_handle(torch)

    def run():
        _lib.check(L.lrcvt_region_adjacency(nx, ny, nz, site_of.data_ptr(), eng.comp.data_ptr(), S, cap,
                                            edges.data_ptr(), ctypes.byref(got), st), "adjacency")

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"edges": int(got.value), "device_ms": ms, "voxels_per_s": grid.size / (ms / 1e3),
            "algorithmic_GBps": 8.0 * grid.size / (ms / 1e3) / 1e9,
            "note": "lrcvt_region_adjacency: face scan of site_of + component (8 B/voxel), hash-set dedup, sort"}


def one_off_passes(grid, labels, eng, config, S, reps=3):
    """Device-resident timing of the passes reported beside the iteration
    metric: isoband + component masks, and the per-cell
    aggregation (3 field pairs' moments + 64-bin histograms of f and g)."""
    import ctypes

    import torch

    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.pipeline import cell_aggregates_device

    L = _lib.lib()
    st = _lib.stream_handle(torch)
    n = grid.size
    nx, ny, nz = grid.dims
    f = torch.from_numpy(grid.fields["f"]).cuda()
    g = torch.from_numpy(grid.fields["g"]).cuda()
    iso = torch.tensor(CONFIGS[config]["iso"], dtype=torch.float64, device="cuda")
    layer = torch.empty(n, dtype=torch.int32, device="cuda")
    comp = torch.empty(n, dtype=torch.int32, device="cuda")
    nc = ctypes.c_int32()

    def masks():
        _lib.check(L.lrcvt_isobands(n, f.data_ptr(), iso.data_ptr(), iso.numel(), layer.data_ptr(), st), "iso")
        _lib.check(L.lrcvt_label_components(nx, ny, nz, layer.data_ptr(), iso.numel() - 1, comp.data_ptr(),
                                            ctypes.byref(nc), st), "ccl")

    ss_site = eng.ss[:, 0].contiguous()
    pair_idx = np.array([[0, 0], [0, 1], [1, 1]], np.int32)

    def agg():
        cell_aggregates_device([f, g], eng.comp, ss_site, S, labels.n_components, pair_idx, bins=64)

    out = {}
    for name, fn, bytes_per_voxel in (("masks", masks, 8 + 12), ("aggregate", agg, 16)):
        fn()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(reps):
            fn()
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / reps
        out[name] = {"ms": ms, "voxels_per_s": n / (ms / 1e3),
                     "algorithmic_GBps": bytes_per_voxel * n / (ms / 1e3) / 1e9}
    out["masks"]["note"] = "isobands (f32 read + i32 write) + 6-conn CCL with dense ids; bytes counted 20/voxel"
    out["aggregate"]["note"] = ("per-cell n, 15 power sums x 3 pairs, min/max, 64-bin hist of f and g; "
                                "16 B/voxel (f, g, site_of, component)")
    return out


def cpu_baseline(grid, labels, params, weights, pos, sc, budget_s=45.0, max_iters=3):
    from oracle import oracle

    oracle.build()
    oracle.set_num_threads(os.cpu_count() or 1)
    w = None if params.weight_field is None else weights
    comp = labels.component
    t0 = time.perf_counter()
    it = 0
    p = pos
    while it < max_iters and (it == 0 or time.perf_counter() - t0 < budget_s):
        c = oracle.classify(grid.dims, grid.spacing, comp, p, sc, labels.n_components)
        p = oracle.centroidal(grid.dims, grid.spacing, comp, c["site_of"], c["src"], w, p, sc)["new_pos"]
        it += 1
    dt = time.perf_counter() - t0
    return {"value": grid.size * it / dt, "unit": "voxels/s", "cores": oracle.num_threads(), "kind": "port",
            "sample": f"{it} Lloyd iteration(s) of the same workload from the timed region's starting sites"}


def run_global(args, cfg, world, rank, local):
    """--mode global: ONE volume split into z-slabs (paper_2208_06970_b200.multigpu):
    each rank evaluates, commits and votes over its own slab; boundary-plane
    proposals go to the neighbour ranks, far reads through peer pointers
    (CUDA IPC / NVLink P2P). value = voxels x steps / max-over-ranks device
    time (strong scaling). With one process, --emulate-ranks K runs K slab
    ranks on this GPU one after another and reports each rank's own device
    time per iteration (the slowest bounds what K GPUs would take)."""
    import torch

    from paper_2208_06970_b200.multigpu import Emulated, GlobalClassifier, TorchDist
    from paper_2208_06970_b200.tessellation import lloyd_weight_mode, voxel_length

    grid, labels, params, sites, weights = build_workload(cfg, 0)
    emulate = world == 1 and args.emulate_ranks > 1
    coll = TorchDist() if world > 1 else Emulated(max(1, args.emulate_ranks))
    S = len(sites)
    gc = GlobalClassifier(grid.dims, grid.spacing, labels.component, labels.n_components, S, coll)
    pos_d = torch.from_numpy(np.array([s.position for s in sites])).cuda()
    sc_d = torch.from_numpy(np.array([s.component_id for s in sites], np.int32)).cuda()
    mode, w_d = lloyd_weight_mode(torch, grid, params, weights)
    vlen = voxel_length(grid.dims, grid.spacing)
    inband = int(gc.any_engine().inband)

    last = {}

    def step(p):
        last.update(gc.classify(p, sc_d))
        p2, _, _ = gc.centroidal(p, sc_d, mode, w_d, 0.5 * vlen)
        return p2

    gc.reuse_sites(True)  # Lloyd loop: site components fixed
    for _ in range(args.warmup):
        pos_d = step(pos_d)
    bounds0 = list(gc.bounds)
    if not args.no_rebalance:
        # slab bounds from measured per-rank device time: twice, a calibration iteration (not timed) and a
        # re-cut; then one more warm-up iteration on the final bounds
        for _ in range(2):
            gc.set_timing(True)
            gc.rank_ms()
            pos_d = step(pos_d)
            cost = gc.rank_ms()
            gc.set_timing(False)
            gc.rebalance(cost)
        pos_d = step(pos_d)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    gc.set_timing(emulate)
    gc.rank_ms()
    gc.calls = {r: {} for r in gc.engines}
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LRCVT_BENCH_DEVICE", local))) as clk:
        t0.record()
        for _ in range(args.steps):
            pos_d = step(pos_d)
        t1.record()
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    per_cat = gc.rank_ms(breakdown=True) if emulate else None
    per_rank = {r: sum(c.values()) for r, c in per_cat.items()} if emulate else None
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        line = {
            "metric": "CVT-iteration voxels/s", "value": grid.size * args.steps / (ms / 1e3), "unit": "voxels/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "mode": "global", "slabs": coll.world,
            "config": bench_config(cfg, grid.size, S, inband), "clocks": clk.summary(),
            "counters": {k: last[k] for k in ("rounds", "sweeps", "evaluations", "commits") if k in last},
            "slabs_z": [list(b) for b in gc.bounds], "slabs_z_inband_balanced": [list(b) for b in bounds0]}
        if emulate:
            slow = max(per_rank.values()) / args.steps
            line["emulated_ranks"] = {
                "ranks": coll.world, "rank_ms_per_step": {str(r): v / args.steps for r, v in per_rank.items()},
                "slowest_rank_ms_per_step": slow,
                "slowest_rank_breakdown_ms_per_step": {
                    k: v / args.steps for k, v in per_cat[max(per_rank, key=per_rank.get)].items()},
                "slowest_rank_calls_per_step": {
                    k: v / args.steps for k, v in gc.calls[max(per_rank, key=per_rank.get)].items()},
                "projected_value": grid.size / (slow / 1e3),
                "note": "all slab ranks on ONE GPU one after another; each rank's own kernels timed with CUDA "
                        "events (the host round trips of the per-round count reads excluded; collectives are host "
                        "list operations here, so NVLink transfer time is not included); `value` above is the "
                        "serial sum over ranks"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with one rank per GPU on 127.0.0.1."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd)


def e2e_public_api(grid, labels, params, weights, pos_start, sc_np, steps, world):
    """End to end through the public API, honouring the reference's output
    contract: per step voronoi_classify(grid, labels, sites, weights) with host
    Site lists in, the four per-voxel arrays materialised as numpy
    (site_of/dist/src/state, tessellation.py:120-122, :205-208), then
    centroidal_update(tess) with host Site lists out. Also the same loop
    without reading the arrays (they stay in HBM; `lazy`)."""
    import torch

    from paper_2208_06970_b200 import centroidal_update, voronoi_classify
    from paper_2208_06970_b200.seeding import Site

    n, S = grid.size, len(sc_np)
    w = weights if params.weight_field else None

    def run(k, full):
        cur = [Site(tuple(p), int(c)) for p, c in zip(pos_start, sc_np)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            t_ = voronoi_classify(grid, labels, cur, w)
            if full:
                _ = (t_.site_of, t_.dist, t_.src, t_.state)
            cur, _ = centroidal_update(t_)
            del t_
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    run(2, True)  # warm-up: plans, graphs, pinned host pool
    ke = max(1, min(steps, 10))
    dt_full = run(ke, True)
    dt_lazy = run(ke, False)
    h2d = 2 * S * (24 + 4)
    d2h_small = S * (24 + 8) + 64
    return {"value": n * ke * world / dt_full, "unit": "voxels/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h_small + n * (4 + 8 + 4 + 1), "steps": ke,
            "note": "public API per step: voronoi_classify(grid, labels, sites, weights) + reading tess.site_of/"
                    "dist/src/state as numpy (the reference's Tessellation output) + centroidal_update(tess); "
                    "host Site lists in and out; labels/weights uploaded once",
            "lazy": {"value": n * ke * world / dt_lazy, "unit": "voxels/s", "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h_small,
                     "note": "same loop without reading the per-voxel arrays (they stay in HBM)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-budget", type=float, default=420.0,
                    help="--impl reference: seconds of timed CPU work before the sample stops")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-passes", action="store_true")
    ap.add_argument("--no-rebalance", action="store_true",
                    help="--mode global: keep the in-band-balanced slab bounds (no calibration iteration)")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="--mode global on one process: run this many z-slab ranks on the one GPU")
    ap.add_argument("--mode", default=None, choices=["blocks", "global"],
                    help="global (default for N > 1): one volume z-slab partitioned over the ranks (strong "
                         "scaling); blocks: one independent volume per rank (weak scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world, rank, local = dist_setup(args)
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    args.mode = args.mode or ("global" if world > 1 else "blocks")
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import torch

    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.tessellation import engine_for, lloyd_weight_mode, voxel_length

    # LRCVT_BENCH_DEVICE / LRCVT_BENCH_BACKEND exist only to smoke-test the multi-rank code path on a
    # one-GPU box (ranks sharing device 0 over gloo; block-mode ranks never wait on each other's kernels)
    dev_index = int(os.environ.get("LRCVT_BENCH_DEVICE", local))
    torch.cuda.set_device(dev_index)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("LRCVT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    if args.mode == "global" and (world > 1 or args.emulate_ranks > 1):
        run_global(args, cfg, world, rank, local)
        return
    grid, labels, params, sites, weights = build_workload(cfg, rank)
    n = grid.size
    S = len(sites)
    L = _lib.lib()
    eng = engine_for(labels, grid.spacing, S)
    pos0 = np.array([s.position for s in sites])
    sc_np = np.array([s.component_id for s in sites], np.int32)
    pos_d = torch.from_numpy(pos0).cuda()
    sc_d = torch.from_numpy(sc_np).cuda()
    mode, w_d = lloyd_weight_mode(torch, grid, params, weights)
    backoff = 0.5 * voxel_length(grid.dims, grid.spacing)
    config = bench_config(cfg, n, S, eng.inband)
    flush = config["l2"].startswith("flushed")
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda") if flush else None

    def step(p):
        eng.classify(p, sc_d, want_state=True)
        p2, disp, _, _ = eng.centroidal(p, sc_d, mode, w_d, backoff)
        return p2, disp

    L.lrcvt_plan_reuse_eligible(eng.plan, 2)  # Lloyd loop: site components fixed from its first classify
    for _ in range(args.warmup):
        pos_d, _ = step(pos_d)
    torch.cuda.synchronize()
    pos_start = pos_d.cpu().numpy()

    # timed region: device-side round loops (CUDA graphs), no per-launch events
    E = C = R = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = L.lrcvt_launch_count()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(int(os.environ.get("LRCVT_BENCH_DEVICE", local))) as clk:
        for k in range(args.steps):
            if flush:
                scratch.zero_()
            ev[k][0].record()
            pos_d, _ = step(pos_d)
            ev[k][1].record()
            st = eng.stats
            E += st.evaluations
            C += st.commits
            R += st.rounds
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = int(L.lrcvt_launch_count() - launches0)
    ms = sum(a.elapsed_time(b) for a, b in ev)
    # breakdown / dominant-kernel pass: the same K iterations replayed from the
    # timed region's starting sites with host-driven rounds and CUDA events
    # around every eval and commit launch (not part of the timed number)
    _lib.check(L.lrcvt_plan_set_timing(eng.plan, 1), "set_timing")
    pos_b = torch.from_numpy(pos_start).cuda()
    for k in range(args.steps):
        if flush:
            scratch.zero_()
        pos_b, _ = step(pos_b)
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64,
                         device="cuda" if torch.distributed.get_backend() == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    el, eitems, ems = _lib.ctypes.c_int64(), _lib.ctypes.c_int64(), _lib.ctypes.c_double()
    L.lrcvt_plan_timing(eng.plan, _lib.ctypes.byref(el), _lib.ctypes.byref(eitems), _lib.ctypes.byref(ems))
    prof = (_lib.ctypes.c_double * 6)()
    L.lrcvt_plan_profile(eng.plan, prof)
    _lib.check(L.lrcvt_plan_set_timing(eng.plan, 0), "set_timing")
    value = n * args.steps * world / (ms / 1e3)
    hbm, peak_kind = peaks()
    clocks = clk.summary()
    # dominant kernel: k_eval; algorithmic bytes = 20 B per evaluated voxel
    eval_bytes = 20.0 * eitems.value
    achieved = eval_bytes / (ems.value / 1e3) / 1e9 if ems.value > 0 else 0.0
    b_iter = 29.0 * n + 20.0 * E / args.steps + 16.0 * C / args.steps
    traffic = issue = None
    prof_path = ROOT / "profiles" / f"ncu_{args.config}_k_eval.json"
    if prof_path.exists() and el.value:
        pj = json.loads(prof_path.read_text())
        if pj.get("dram_bytes_per_item"):
            traffic = pj["dram_bytes_per_item"] * eitems.value / el.value
        # issue roof: warp instructions the eval launches execute (ncu, per evaluated voxel) over what 148 SMs x
        # 4 schedulers issue in the measured eval time at the sampled SM clock
        if pj.get("warp_inst_per_item") and clocks.get("sm_mhz"):
            inst = pj["warp_inst_per_item"] * eitems.value
            issue = {"warp_inst_per_item": pj["warp_inst_per_item"],
                     "frac": inst / (148 * 4 * clocks["sm_mhz"] * 1e6 * ems.value / 1e3)}

    L.lrcvt_plan_reuse_eligible(eng.plan, 0)  # public-API e2e below takes the general path
    passes = one_off_passes(grid, labels, eng, args.config, S) if not args.no_passes else None
    if passes is not None:
        passes["seeding"] = seeding_pass(grid, labels, params)
        passes["layout"] = layout_pass(grid, labels, eng, S)
        passes["adjacency"] = adjacency_pass(grid, eng, S)
    e2e = None if args.no_e2e else e2e_public_api(grid, labels, params, weights, pos_start, sc_np, args.steps,
                                                  world)

    line = {
        "metric": "CVT-iteration voxels/s", "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "counters": {"E_per_step": E / args.steps, "C_per_step": C / args.steps, "rounds_per_step": R / args.steps},
        "roofline": {"bound": "hbm", "kernel": "k_eval", "achieved": achieved, "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "issue": issue,
                     "launches": el.value, "avg_launch_us": 1e3 * ems.value / max(el.value, 1),
                     "bytes_per_launch": eval_bytes / max(el.value, 1),
                     "eval_share_of_step": ems.value / ms if ms else None,
                     "breakdown_ms_per_step": {"eval_phase1": prof[0] / args.steps,
                                               "eval_phase2": prof[1] / args.steps,
                                               "commit": prof[2] / args.steps},
                     "iteration_B": b_iter, "iteration_frac": b_iter / (ms / args.steps / 1e3) / 1e9 / hbm},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if e2e:
        line["e2e"] = e2e
    if passes:
        line["passes"] = passes
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(grid, labels, params, weights, pos_start, sc_np)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

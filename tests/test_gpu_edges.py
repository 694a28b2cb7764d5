"""GPU edge cases against the CPU oracle (bit-exact): degenerate grids,
contested seed voxels, components without sites, non-power-of-two spacing in
3D, many small components, early Lloyd stop."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _labels(comp, dims):
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap

    comp = np.ascontiguousarray(comp, dtype=np.int32)
    n = int(comp.max()) + 1 if (comp >= 0).any() else 0
    counts = np.bincount(comp[comp >= 0], minlength=n)
    table = [ComponentInfo(c, 0, int(counts[c]), (0,) * 6, (0.0, 1.0)) for c in range(n)]
    return LabelMap(tuple(dims), np.where(comp >= 0, 0, -1).astype(np.int32), comp, table, [0.0, 1.0], "f")


def _check(grid, labels, sites, oracle, weights=None):
    from paper_2208_06970_b200 import centroidal_update, voronoi_classify

    tess = voronoi_classify(grid, labels, sites, weights)
    pos, sc = tess.site_positions(), tess.site_components()
    ref = oracle.classify(grid.dims, grid.spacing, labels.component, pos, sc, labels.n_components)
    for k in ("site_of", "dist", "src", "state"):
        assert np.array_equal(getattr(tess, k), ref[k]), k
    assert tess.report["rounds"] == ref["rounds"] and tess.report["sweeps"] == ref["sweeps"]
    new_sites, mean_ds = centroidal_update(tess)
    u = oracle.centroidal(grid.dims, grid.spacing, labels.component, ref["site_of"], ref["src"], weights, pos, sc)
    assert np.array_equal(np.array([s.position for s in new_sites]).reshape(-1, 3), u["new_pos"])
    assert mean_ds == u["mean_ds"]
    assert tess.report["empty_regions"] == u["empty"]
    return tess


def test_single_voxel_grid(oracle_mod):
    from paper_2208_06970_b200 import Site, VoxelGrid

    grid = VoxelGrid((1, 1, 1), (1, 1, 1), {})
    _check(grid, _labels(np.zeros(1), (1, 1, 1)), [Site((0.3, 0.7, 0.5), 0)], oracle_mod)


def test_long_line_grid(oracle_mod):
    from paper_2208_06970_b200 import Site, VoxelGrid

    n = 5000
    grid = VoxelGrid((n, 1, 1), (1, 1, 1), {})
    comp = np.zeros(n, np.int32)
    comp[2000:2100] = -1  # a gap splits the line into two components
    comp[2100:] = 1
    sites = [Site((10.5, 0.5, 0.5), 0), Site((1500.25, 0.5, 0.5), 0), Site((4999.5, 0.5, 0.5), 1)]
    _check(grid, _labels(comp, (n, 1, 1)), sites, oracle_mod)


def test_contested_seed_voxels_and_empty_regions(oracle_mod):
    """Several sites in one voxel: the lexicographic (distance, id) winner
    takes the voxel, the others keep empty regions and do not move."""
    from paper_2208_06970_b200 import Site, VoxelGrid

    dims = (24, 20, 6)
    grid = VoxelGrid(dims, (1, 1, 1), {})
    comp = np.zeros(int(np.prod(dims)), np.int32)
    sites = [Site((5.5, 5.5, 2.5), 0), Site((5.2, 5.9, 2.1), 0), Site((5.5, 5.5, 2.5), 0),
             Site((17.9, 12.1, 3.3), 0), Site((17.1, 12.9, 3.9), 0)]
    tess = _check(grid, _labels(comp, dims), sites, oracle_mod)
    assert tess.report["empty_regions"] >= 1


def test_large_seed_collision_groups(oracle_mod):
    """2600 sites in three voxels (exact duplicates and jittered positions:
    distance ties inside EPS): the sort-free seed placement folds each group
    in increasing site id over a multi-pass bitonic sort of the collisions."""
    from paper_2208_06970_b200 import Site, VoxelGrid

    dims = (16, 16, 4)
    grid = VoxelGrid(dims, (1, 1, 1), {})
    comp = np.zeros(int(np.prod(dims)), np.int32)
    rng = np.random.default_rng(7)
    cells = [(3, 3, 1), (9, 4, 0), (12, 12, 2)]
    sites = []
    for i in range(2600):
        c = cells[i % 3]
        if i % 5 == 0:
            p = (c[0] + 0.5, c[1] + 0.5, c[2] + 0.5)
        else:
            p = (c[0] + rng.random(), c[1] + rng.random(), c[2] + rng.random())
        sites.append(Site(p, 0))
    tess = _check(grid, _labels(comp, dims), sites, oracle_mod)
    assert tess.report["empty_regions"] >= 2597


def test_components_without_sites_and_many_components(oracle_mod):
    from paper_2208_06970_b200 import (IsobandSpec, Site, VoxelGrid, classify_isobands, label_components)

    rng = np.random.default_rng(4)
    dims = (40, 30, 20)
    f = rng.random(int(np.prod(dims))).astype(np.float32)
    grid = VoxelGrid(dims, (1, 1, 1), {"f": f})
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.2, 0.6])))
    assert labels.n_components > 100
    nx, ny = dims[0], dims[1]
    sites = []
    for c in labels.component_table[::7][:60]:
        v = int(np.flatnonzero(labels.component == c.id)[0])
        sites.append(Site(((v % nx) + 0.25, ((v // nx) % ny) + 0.75, (v // (nx * ny)) + 0.5), c.id))
    tess = _check(grid, labels, sites, oracle_mod)
    assert len(tess.report["components_without_sites"]) == labels.n_components - len(sites)


def test_non_dyadic_spacing_3d(oracle_mod):
    from paper_2208_06970_b200 import IsobandSpec, SeedingParams, VoxelGrid, classify_isobands, label_components
    from paper_2208_06970_b200 import seed_sites, synth_field, voxel_weights

    base = synth_field("random-smooth", (30, 26, 22), 5)
    grid = VoxelGrid(base.dims, (0.7, 1.3, 0.45), base.fields)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.3, 0.6, 0.85])))
    params = SeedingParams(alpha=50, seed=2, weight_field="g", gamma=1.5)
    sites, _ = seed_sites(grid, labels, params)
    _check(grid, labels, sites, oracle_mod, voxel_weights(grid, params))


def test_lloyd_tolerance_stops_early():
    from paper_2208_06970_b200 import LloydParams, SeedingParams, VoxelGrid, lrcvt

    f = np.full(15 * 15, 0.5, np.float32)
    grid = VoxelGrid((15, 15, 1), (1, 1, 1), {"f": f})
    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components

    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.0, 1.0])))
    _, trace = lrcvt(grid, labels, SeedingParams(alpha=4, seed=1), LloydParams(max_updates=50, ds_tolerance=0.5))
    assert len(trace) < 50 and trace[-1] < 0.5


def test_zero_sites():
    from paper_2208_06970_b200 import VoxelGrid, voronoi_classify

    grid = VoxelGrid((4, 4, 1), (1, 1, 1), {})
    tess = voronoi_classify(grid, _labels(np.zeros(16), (4, 4, 1)), [])
    assert np.all(tess.site_of == -1) and np.all(np.isinf(tess.dist))
    assert tess.report["components_without_sites"] == [0]


@pytest.mark.parametrize("spacing", [(1.0, 1.0, 1.0), (0.7, 1.3, 2.1)])
def test_labyrinth_thin_walls_and_thick_chambers(spacing, oracle_mod):
    """Thick chambers (clearance shortcut proves most rays) separated by
    one-voxel walls with pinholes (rays graze walls and thread the holes):
    exercises the clearance bound, the strict-order rule and the exact
    fallbacks against the oracle, in dyadic and non-dyadic spacing."""
    from paper_2208_06970_b200 import Site, VoxelGrid

    dims = (56, 44, 36)
    nx, ny, nz = dims
    comp = np.zeros((nz, ny, nx), np.int32)
    comp[:, :, 18] = -1
    comp[:, :, 37] = -1
    comp[:, 20, :] = -1
    comp[17, :, :] = -1
    rng = np.random.default_rng(11)
    for _ in range(40):  # pinholes through the walls
        z, y = rng.integers(1, nz - 1), rng.integers(1, ny - 1)
        comp[z, y, rng.choice([18, 37])] = 0
        comp[rng.integers(1, nz - 1), 20, rng.integers(1, nx - 1)] = 0
        comp[17, rng.integers(1, ny - 1), rng.integers(1, nx - 1)] = 0
    comp = comp.reshape(-1)
    grid = VoxelGrid(dims, spacing, {})
    labels = _labels(comp, dims)
    sx, sy, sz = spacing
    sites = []
    for _ in range(70):
        while True:
            x, y, z = rng.integers(0, nx), rng.integers(0, ny), rng.integers(0, nz)
            if comp[x + nx * (y + ny * z)] == 0:
                break
        sites.append(Site(((x + rng.random()) * sx, (y + rng.random()) * sy, (z + rng.random()) * sz), 0))
    _check(grid, labels, sites, oracle_mod)


@pytest.mark.parametrize("kind,dims,iso,spacing", [
    ("random-smooth", (48, 40, 36), [0.35, 0.5, 0.65, 0.8], (1.0, 1.0, 1.0)),
    ("horseshoe", (40, 40, 32), [0.0, 0.12, 0.3], (1.0, 0.5, 2.0)),
    ("spiral", (64, 64, 1), [0.3, 0.55, 0.8], (1.0, 1.0, 1.0)),
])
def test_clearance_dda_equals_reference_dda(kind, dims, iso, spacing):
    """The eval kernels' ray test (segment_clear_fast: the reference DDA plus
    the static-clearance shortcuts) agrees with the plain DDA
    (_segment_hit_t >= 1, itself pinned to the reference's ray golden) on
    random segments between in-band points, long and short."""
    import torch

    from paper_2208_06970_b200 import IsobandSpec, classify_isobands, label_components, synth_field
    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.grid import VoxelGrid
    from paper_2208_06970_b200.tessellation import engine_for, segment_hit_t_batch

    g0 = synth_field(kind, dims, 1)
    grid = VoxelGrid(dims, spacing, g0.fields)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", iso)))
    eng = engine_for(labels, spacing, 1)
    rng = np.random.default_rng(4)
    inb = np.flatnonzero(labels.component >= 0)
    n = 60000
    nx, ny, nz = dims
    v = rng.choice(inb, n)
    a = np.stack([v % nx + rng.random(n), (v // nx) % ny + rng.random(n), v // (nx * ny) + rng.random(n)], 1)
    span = np.where(rng.random(n) < 0.5, 4.0, 40.0)[:, None]
    b = a + (rng.random((n, 3)) - 0.5) * 2 * span
    if nz == 1:
        a[:, 2] = 0.5
        b[:, 2] = 0.5
    a *= spacing
    b *= spacing
    segs = np.ascontiguousarray(np.concatenate([a, b], 1))
    want = labels.component[v].astype(np.int32)
    t = segment_hit_t_batch(labels, segs, want, spacing)
    L = _lib.lib()
    segs_d = torch.from_numpy(segs).cuda()
    want_d = torch.from_numpy(want).cuda()
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.check(L.lrcvt_segment_clear_batch(eng.plan, segs_d.data_ptr(), want_d.data_ptr(), n, out.data_ptr(),
                                           _lib.stream_handle(torch)), "clear batch")
    fast = out.cpu().numpy().astype(bool)
    assert np.array_equal(fast, t >= 1.0)
    assert 0.05 < fast.mean() < 0.95  # both outcomes well represented


def test_reuse_run_rebuilds_eligible_list_for_new_sites(oracle_mod):
    """A Lloyd-style run (lrcvt_plan_reuse_eligible(plan, 2)) on an engine whose
    last classify had other site components but the same site count builds
    its own eligible list instead of reusing the stale one."""
    import torch

    from paper_2208_06970_b200 import Site, VoxelGrid, voronoi_classify
    from paper_2208_06970_b200.tessellation import engine_for

    dims = (20, 16, 6)
    grid = VoxelGrid(dims, (1, 1, 1), {})
    comp = np.zeros(int(np.prod(dims)), np.int32)
    comp.reshape(6, 16, 20)[:, :, 10:] = 1  # two components side by side
    labels = _labels(comp, dims)
    a = [Site((2.5, 3.5, 2.5), 0), Site((6.5, 9.5, 3.5), 0)]  # component 0 only
    b = [Site((2.5, 3.5, 2.5), 0), Site((15.5, 9.5, 3.5), 1)]  # both components, same count
    voronoi_classify(grid, labels, a)  # the shared engine now holds a's eligible list
    eng = engine_for(labels, grid.spacing, len(b))
    pos = torch.tensor([s.position for s in b], dtype=torch.float64).cuda()
    sc = torch.tensor([s.component_id for s in b], dtype=torch.int32).cuda()
    eng.L.lrcvt_plan_reuse_eligible(eng.plan, 2)
    try:
        eng.classify(pos, sc, want_state=True)
    finally:
        eng.L.lrcvt_plan_reuse_eligible(eng.plan, 0)
    ref = oracle_mod.classify(dims, (1.0, 1.0, 1.0), comp, pos.cpu().numpy(), sc.cpu().numpy(), 2)
    assert np.array_equal(eng.ss[:, 0].cpu().numpy(), ref["site_of"])
    assert np.array_equal(eng.state.cpu().numpy(), ref["state"])

"""Host side of the public API (CPU): the C builder of list[Site]
(csrc/sites_ext.c) gives the objects the reference's Python loop builds, and
the cached site arrays follow every change a caller can make to the list."""

import numpy as np


def test_c_site_builder_matches_python():
    from paper_2208_06970_b200 import tessellation as T
    from paper_2208_06970_b200.seeding import Site

    assert T._sites is not None, "build() compiles paper_2208_06970_b200/_sites*.so"
    rng = np.random.default_rng(3)
    pos = rng.random((1000, 3)) * 512
    comp = rng.integers(-1, 50, 1000).astype(np.int32)
    got = T.make_sites(pos, comp)
    want = [Site((float(p[0]), float(p[1]), float(p[2])), int(c)) for p, c in zip(pos, comp)]
    assert got == want
    assert all(type(s) is Site and type(s.position) is tuple and type(s.component_id) is int for s in got)
    assert all(type(x) is float for s in got[:20] for x in s.position)
    got[5].position = (1.0, 2.0, 3.0)  # an ordinary mutable dataclass instance
    assert got[5].position == (1.0, 2.0, 3.0)
    assert T.make_sites(np.zeros((0, 3)), np.zeros(0, np.int32)) == []


def test_cached_site_arrays_follow_changes():
    from paper_2208_06970_b200 import tessellation as T
    from paper_2208_06970_b200.seeding import Site

    pos = np.arange(15, dtype=np.float64).reshape(5, 3)
    comp = np.arange(5, dtype=np.int32)
    sites = T.make_sites(pos, comp)
    assert np.array_equal(T._positions(sites), pos) and np.array_equal(T._components(sites), comp)
    sites[2].position = (9.0, 9.0, 9.0)
    assert T._positions(sites)[2].tolist() == [9.0, 9.0, 9.0]
    sites[1] = Site((1.0, 2.0, 3.0), 7)
    assert T._components(sites)[1] == 7 and T._positions(sites)[1].tolist() == [1.0, 2.0, 3.0]
    sites[3].component_id = 42
    assert T._components(sites)[3] == 42
    copy = list(sites)  # another list holding the same objects
    assert np.array_equal(T._positions(copy), T._positions(sites))
    out = T._positions(sites)
    out[0] = -1.0  # callers get copies
    assert T._positions(sites)[0, 0] == 0.0

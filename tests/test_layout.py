"""The .lrcvt layout (layout.py:123-488 of the reference; SURVEY.md §8(f)
rank 2) against files the reference itself wrote (tests/golden/layout.json:
sha256 of the whole file, of the record block and of the manifest).

CPU: the oracle's record order / index arrays reproduce the reference's record
block, and the product's host assembly (index tables, header, writer,
manifest) turns them into byte-identical files; the reader round-trips them.
GPU: build_and_write with the device record pass gives the same bytes."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def _gold():
    meta = json.loads((GOLD / "layout.json").read_text())
    arr = np.load(GOLD / "layout.npz")
    return meta, arr


def _inputs(name, m, arr):
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap, VoxelGrid
    from paper_2208_06970_b200.layout import AggregateBlob
    from paper_2208_06970_b200.seeding import Site
    from paper_2208_06970_b200.tessellation import Tessellation

    dims = tuple(m["dims"])
    grid = VoxelGrid(dims, tuple(m["spacing"]), {k: arr[f"{name}/field/{k}"] for k in m["fields"]})
    table = [ComponentInfo(t["id"], t["layer"], t["voxel_count"], tuple(t["bbox"]), tuple(t["band"]))
             for t in m["table"]]
    labels = LabelMap(dims, arr[f"{name}/layer"], arr[f"{name}/component"], table, m["iso_values"],
                      m["iso_field"])
    sites = [Site(tuple(s[:3]), int(s[3])) for s in m["sites"]]
    n = int(np.prod(dims))
    z = np.zeros(n)
    tess = Tessellation(dims, grid.spacing, arr[f"{name}/site_of"], z, z.astype(np.int32), z.astype(np.uint8),
                        labels.component, sites)
    blobs = [AggregateBlob(b["scope"], b["id"], b["kind"], b["payload"].encode()) for b in m["blobs"]]
    return grid, labels, tess, blobs


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


CASES = ["explore", "stray", "smooth3d"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_records_match_reference(name, oracle_mod):
    meta, arr = _gold()
    m = meta[name]
    grid, labels, tess, _ = _inputs(name, m, arr)
    rec, _, _, _ = oracle_mod.layout_records(grid.dims, labels.component, tess.site_of,
                                             [grid.fields[k] for k in m["fields"]], labels.n_components)
    assert _sha(rec.tobytes()) == m["data_sha"]


@pytest.mark.parametrize("name", CASES)
def test_host_assembly_byte_identical(name, oracle_mod, tmp_path):
    """Index tables + header + writer + manifest of the product, fed with the
    oracle's record arrays, reproduce the reference's file bytes."""
    from paper_2208_06970_b200 import layout as LY

    meta, arr = _gold()
    m = meta[name]
    grid, labels, tess, blobs = _inputs(name, m, arr)
    rec, key, first, count = oracle_mod.layout_records(grid.dims, labels.component, tess.site_of,
                                                       [grid.fields[k] for k in m["fields"]], labels.n_components)
    layers, comps, regions = LY._index_tables(labels, tess, key.astype(np.uint32), first, count)
    h = LY.Header(grid.dims, grid.spacing, grid.field_names(), labels.field_name, list(labels.iso_values),
                  int(rec.size), layers, comps, regions)
    path = tmp_path / f"{name}.lrcvt"
    LY._write(path, h, rec, blobs)
    assert _sha(path.read_bytes()) == m["file_sha"]
    assert _sha(json.dumps(LY._manifest(h, blobs), indent=1).encode()) == m["manifest_sha"]
    # the reader round-trips the reference-format file
    rd = LY.LayoutReader(path)
    assert rd.header.n_records == rec.size and len(rd.aggregates) == len(blobs)
    assert rd.all_records().tobytes() == rec.tobytes()
    for c in rd.header.components:
        got = rd.component_records(c.id)
        assert got.size == c.record_count
    one = LY.load_component(path, 0)
    assert one["entry"].id == 0


def test_reader_rejects_bad_files(tmp_path):
    from paper_2208_06970_b200.layout import LayoutReader

    p = tmp_path / "bad.lrcvt"
    p.write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(ValueError, match="magic"):
        LayoutReader(p)


def test_reduction_estimate():
    from paper_2208_06970_b200.layout import reduction_estimate

    assert reduction_estimate(100, 40, 2, 1, 3) == 60 * 3 + 4
    with pytest.raises(ValueError):
        reduction_estimate(10, 11, 1, 1, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_layout_byte_identical(name, tmp_path):
    from paper_2208_06970_b200.layout import build_and_write

    meta, arr = _gold()
    m = meta[name]
    grid, labels, tess, blobs = _inputs(name, m, arr)
    path = tmp_path / f"{name}.lrcvt"
    summary = build_and_write(grid, labels, tess, blobs, path)
    assert _sha(path.read_bytes()) == m["file_sha"]
    assert _sha(Path(str(path) + ".manifest.json").read_bytes()) == m["manifest_sha"]
    summary.pop("path")
    assert summary == m["summary"]


@pytest.mark.gpu
def test_gpu_layout_pipeline_vs_oracle(oracle_mod, tmp_path):
    """Fresh volume through the GPU pipeline: the device record pass equals
    the oracle restatement (records, region keys, component ranges)."""
    from paper_2208_06970_b200 import (IsobandSpec, LloydParams, SeedingParams, classify_isobands,
                                       label_components, lrcvt, synth_field)
    from paper_2208_06970_b200.layout import _site_of_device, device_records

    grid = synth_field("gaussian-mix", (40, 36, 28), 0)
    labels = label_components(classify_isobands(grid, IsobandSpec("f", [0.2, 0.45, 0.7])))
    tess, _ = lrcvt(grid, labels, SeedingParams(alpha=60, weight_field="g", seed=1), LloydParams(max_updates=2))
    rec, region, first, count = device_records(grid, labels, _site_of_device(tess), grid.field_names(),
                                               len(tess.sites))
    orec, okey, ofirst, ocount = oracle_mod.layout_records(grid.dims, labels.component, tess.site_of,
                                                           [grid.fields[k] for k in grid.field_names()],
                                                           labels.n_components)
    assert rec.tobytes() == orec.tobytes()
    assert np.array_equal(region.astype(np.uint64), okey)
    assert np.array_equal(first, ofirst) and np.array_equal(count, ocount)

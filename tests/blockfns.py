"""Oracle-backed per-block compute for CPU tests of the block-mode drivers
(test infrastructure: the product drivers default to the GPU kernels)."""

import numpy as np


def oracle_label(sub, iso):
    from oracle import oracle
    from paper_2208_06970_b200.grid import ComponentInfo, LabelMap

    layer = oracle.isobands(sub.fields[iso.field_name], iso.iso_values)
    comp, table = oracle.label_components(layer, sub.dims, iso.n_bands)
    infos = [ComponentInfo(t["id"], t["layer"], t["voxel_count"], tuple(t["bbox"]),
                           (iso.iso_values[t["layer"]], iso.iso_values[t["layer"] + 1])) for t in table]
    return LabelMap(sub.dims, layer, comp, infos, list(iso.iso_values), iso.field_name)


def oracle_lloyd(sub, labels, seeding, lloyd):
    from oracle import oracle
    from paper_2208_06970_b200.seeding import Site, seed_sites, voxel_weights
    from paper_2208_06970_b200.tessellation import Tessellation

    sites, rep = seed_sites(sub, labels, seeding)
    w = voxel_weights(sub, seeding)
    pos = np.array([s.position for s in sites], dtype=np.float64).reshape(-1, 3)
    sc = np.array([s.component_id for s in sites], dtype=np.int32)
    final, trace, hist = oracle.lloyd(sub.dims, sub.spacing, labels.component, labels.n_components, pos, sc,
                                      None if seeding.weight_field is None else w, lloyd.max_updates,
                                      lloyd.ds_tolerance)
    fin_sites = [Site((float(p[0]), float(p[1]), float(p[2])), int(c)) for p, c in zip(hist[-1], sc)]
    t = Tessellation(sub.dims, sub.spacing, final["site_of"], final["dist"], final["src"], final["state"],
                     labels.component, fin_sites, {"seeding": rep, "updates": len(trace)}, w)
    return t, trace

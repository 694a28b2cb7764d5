"""Blend the phase-1 and phase-2 eval summaries of tools/eval_roof.py into the
one per-evaluated-voxel figure bench.py reads (profiles/ncu_<config>_k_eval.json).

The blend weights each phase by the voxels it evaluates per step in the bench
line: phase 2 evaluates the in-band list once per step (plus the small
follow-up rounds its captured launches show), phase 1 the rest of E_per_step.

  python tools/eval_roof_merge.py <p1.json> <p2.json> <bench.json> <config>
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    p1, p2, bench = (json.loads(Path(a).read_text()) for a in sys.argv[1:4])
    cfg = sys.argv[4]
    # the captured phase-2 launches cover whole steps: big launches = steps
    big = [l for l in p2["launches"] if l["items"] >= 0.5 * max(x["items"] for x in p2["launches"])]
    steps = len(big)
    e2 = sum(l["items"] for l in p2["launches"]) / steps
    e = bench["counters"]["E_per_step"]
    e1 = max(e - e2, 0.0)
    out = {}
    for key in ("dram_bytes_per_item", "warp_inst_per_item"):
        out[key] = (e1 * p1[key] + e2 * p2[key]) / (e1 + e2)
    out["phases"] = {
        "phase1": {"items_per_step": e1, "dram_bytes_per_item": p1["dram_bytes_per_item"],
                   "warp_inst_per_item": p1["warp_inst_per_item"], "launches": p1["launches"],
                   "report": p1.get("report")},
        "phase2": {"items_per_step": e2, "dram_bytes_per_item": p2["dram_bytes_per_item"],
                   "warp_inst_per_item": p2["warp_inst_per_item"], "launches": p2["launches"],
                   "report": p2.get("report")},
    }
    out["note"] = ("ncu --set full captures of k_eval_p1 / k_eval_p2 (cold cache per replay, host-driven rounds); "
                   "per-item figures blended by the voxels each phase evaluates per step in the bench line "
                   f"(E_per_step {e:.4g}); bench.py multiplies by evaluated voxels for roofline.traffic / issue")
    p = ROOT / "profiles" / f"ncu_{cfg}_k_eval.json"
    p.write_text(json.dumps(out, indent=1))
    print(json.dumps({k: v for k, v in out.items() if k != "phases"}, indent=1))


if __name__ == "__main__":
    main()

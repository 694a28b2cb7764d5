"""Per-evaluated-voxel DRAM bytes and warp instructions of the eval kernels
from an ncu --set full capture -> profiles/ncu_<config>_k_eval.json, which
bench.py reads for roofline.traffic and roofline.issue.

  python tools/eval_roof.py <report.ncu-rep> <config> [note]
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__grid_size,"
                          "launch__block_size,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    items = dram = inst = 0.0
    launches = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if "k_eval_p" not in name:
            continue
        n = float(r[col["launch__grid_size"]]) * float(r[col["launch__block_size"]])
        b = sum(float(r[col[k]].replace(",", "")) * scale[units[col[k]]]
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        w = float(r[col["smsp__inst_executed.sum"]].replace(",", ""))
        items += n
        dram += b
        inst += w
        launches.append({"kernel": name.split("(")[0], "items": n, "dram_bytes_per_item": b / n,
                         "warp_inst_per_item": w / n})
    out = {"dram_bytes_per_item": dram / items, "warp_inst_per_item": inst / items, "captured_launches": len(launches),
           "launches": launches, "report": Path(rep).name,
           "note": note or "eval launches of an ncu --set full capture (cold cache per replay); items = grid x block "
                           "(the launch's frontier voxels, last tile rounded up); bench.py multiplies by items per "
                           "launch (traffic) and by evaluated voxels (issue roof)"}
    p = ROOT / "profiles" / f"ncu_{cfg}_k_eval.json"
    p.write_text(json.dumps(out, indent=1))
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}, indent=1))


if __name__ == "__main__":
    main()

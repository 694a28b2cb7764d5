"""Turn ncu outputs from a GPU run into the committed profile summaries.

  python tools/profile_summary.py <tag> <launches.csv> <full.ncu-rep> [items_per_launch.json]

Writes profiles/<tag>_launches.csv (the raw per-launch list: device times
are cold-cache and serialised, compare shares), profiles/<tag>_kernel_shares.json
and profiles/<tag>_ncu_full.json (per captured launch: duration, DRAM bytes,
occupancy, issue activity, stall mix) plus profiles/ncu_<config>_k_eval.json
(DRAM bytes per evaluated voxel, read by bench.py for roofline.traffic).
"""

import collections
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in rows[hi + 1:]:
        if len(r) > vi:
            out.append((r[ki].split("(")[0], r[gi], float(r[vi].replace(",", "")) * scale[r[ui]]))
    return out


def shares(ls):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for name, _, us in ls:
        tot[name] += us
        cnt[name] += 1
    total = sum(tot.values())
    return {k: {"launches": cnt[k], "total_us": round(v, 1), "avg_us": round(v / cnt[k], 2),
                "share": round(v / total, 4)} for k, v in sorted(tot.items(), key=lambda x: -x[1])}


def full(rep):
    if str(rep).endswith(".csv"):  # raw page exported on the GPU box (ncu -i rep --page raw --csv)
        out = Path(rep).read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    want = {"grid": "launch__grid_size", "block": "launch__block_size", "regs": "launch__registers_per_thread",
            "duration_us": "gpu__time_duration.sum", "dram_read_B": "dram__bytes_read.sum",
            "dram_write_B": "dram__bytes_write.sum", "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
            "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1_hit_pct": "l1tex__t_sector_hit_rate.pct", "l2_hit_pct": "lts__t_sector_hit_rate.pct",
            "inst_executed": "smsp__inst_executed.sum"}
    units = rows[1]
    res = []
    stall_cols = [(i, n.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, n in enumerate(h)
                  if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k, col in want.items():
            if col in h:
                v = r[h.index(col)].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[h.index(col)]
                if col == "gpu__time_duration.sum":
                    v = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
                if col.startswith("dram__bytes"):
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
                d[k] = v
        st = {n: float(r[i] or 0) for i, n in stall_cols}
        tot = sum(st.values()) or 1.0
        d["stalls"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
        res.append(d)
    return res


def main():
    tag, lcsv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    PROF.mkdir(exist_ok=True)
    shutil.copy(lcsv, PROF / f"{tag}_launches.csv")
    ls = launches(lcsv)
    (PROF / f"{tag}_kernel_shares.json").write_text(json.dumps(shares(ls), indent=1))
    fl = full(rep)
    (PROF / f"{tag}_ncu_full.json").write_text(json.dumps(fl, indent=1))
    if len(sys.argv) > 4:
        # items evaluated by each captured eval launch = threads of the grid that had work:
        # grid * block is an upper bound; the exact counts come from the bench's timing
        # (E / launches), recorded alongside.
        meta = json.loads(Path(sys.argv[4]).read_text())
        ev = [d for d in fl if d["kernel"].startswith("void lrcvt::k_eval") or "k_eval" in d["kernel"]]
        tot_b = sum(d["dram_read_B"] + d["dram_write_B"] for d in ev)
        tot_items = sum(d["grid"] * d["block"] for d in ev)
        (PROF / f"ncu_{meta['config']}_k_eval.json").write_text(json.dumps({
            "dram_bytes_per_item": tot_b / max(tot_items, 1), "captured_launches": len(ev),
            "note": "DRAM read+write bytes per list item over the captured eval launches (ncu --set full, "
                    "cold cache); bench.py multiplies by items per launch for roofline.traffic"}, indent=1))
    for k, v in list(shares(ls).items())[:8]:
        print(f"{k[:50]:50s} {v}")
    for d in fl:
        print({k: d[k] for k in ("kernel", "grid", "duration_us", "dram_read_B", "dram_write_B", "issue_active_pct") if k in d})


if __name__ == "__main__":
    main()

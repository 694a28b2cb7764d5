"""Per-launch summary of an ncu --set full report: device time, DRAM bytes,
achieved DRAM GB/s and its fraction of the measured HBM copy peak, FP64 pipe
utilisation, warps active, registers, stall mix. Writes JSON (+ prints a table).

  python tools/ncu_kernel_table.py <report.ncu-rep> <out.json> [note]
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
           "smsp__average_warp_latency_issue_stalled_wait.ratio"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "second": 1.0}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]

    def val(r, k):
        i = col.get(k)
        if i is None or r[i] == "":
            return None
        v = float(r[i].replace(",", ""))
        return v * SCALE.get(units[i], 1.0)

    launches = []
    for r in rows[2:]:
        t = val(r, "gpu__time_duration.sum")
        rd, wr = val(r, "dram__bytes_read.sum") or 0.0, val(r, "dram__bytes_write.sum") or 0.0
        d = {"kernel": r[col["Kernel Name"]].split("(")[0].replace("void ", ""), "time_ms": t * 1e3,
             "dram_bytes": rd + wr, "dram_GBps": (rd + wr) / t / 1e9, "dram_frac_of_measured_peak": (rd + wr) / t / 1e9 / peak}
        for k, short in (("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
                         ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
                         ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
                         ("sm__inst_executed.sum", "warp_inst"),
                         ("launch__registers_per_thread", "registers"), ("launch__grid_size", "grid"),
                         ("launch__block_size", "block"), ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
                         ("smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio", "stall_long_scoreboard"),
                         ("smsp__average_warp_latency_issue_stalled_wait.ratio", "stall_wait")):
            d[short] = val(r, k)
        launches.append(d)
    Path(out).write_text(json.dumps({"report": Path(rep).name, "note": note, "hbm_peak_GBps_measured": peak,
                                     "launches": launches}, indent=1))
    print(f"{'kernel':40s} {'ms':>8s} {'GB':>7s} {'GB/s':>8s} {'frac':>6s} {'fp64%':>6s} {'warps%':>6s} {'regs':>5s}")
    for d in launches:
        print(f"{d['kernel'][:40]:40s} {d['time_ms']:8.3f} {d['dram_bytes'] / 1e9:7.3f} {d['dram_GBps']:8.1f} "
              f"{d['dram_frac_of_measured_peak']:6.3f} {d['fp64_pipe_pct'] or 0:6.1f} {d['warps_active_pct'] or 0:6.1f} "
              f"{int(d['registers'] or 0):5d}")


if __name__ == "__main__":
    main()

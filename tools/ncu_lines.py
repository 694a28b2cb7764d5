"""Per-CUDA-source-line totals (warp-stall samples, warp instructions) from an
ncu report captured with --import-source on: python tools/ncu_lines.py rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = ""
hdr = None
acc = {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" and len(r) > 3:
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) != len(hdr):
        continue
    try:
        samp = float(r[4] if r[4] not in ("-", "") else 0)
        inst = float(r[7] if r[7] not in ("-", "") else 0)
    except ValueError:
        continue
    a = acc.setdefault((cur_file, int(r[0])), [0.0, 0.0, r[1]])
    a[0] += samp
    a[1] += inst
tot_s = sum(v[0] for v in acc.values()) or 1
tot_i = sum(v[1] for v in acc.values()) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
for (f, ln), (s_, i, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s_ / tot_s:6.3f} {i / tot_i:6.3f}  {f}:{ln:<4} {src.strip()[:90]}")

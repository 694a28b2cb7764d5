"""Per-source-line warp-instruction and stall-sample shares, plus the SASS
opcode mix, of one kernel in an ncu report (--import-source on, -lineinfo).

  python tools/ncu_src_breakdown.py <rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, acc, sass, f = None, None, {}, {}, "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        try:
            cur = (f, int(r[0]), r[1][:90])
        except ValueError:
            pass
        continue
    try:
        inst, samp = float(r[7]), float(r[4])
    except (ValueError, IndexError):
        continue
    a = acc.setdefault(cur, [0.0, 0.0])
    a[0] += inst
    a[1] += samp
    t = r[3].strip().split()
    if t:
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        sass[op] = sass.get(op, 0.0) + inst
tot = sum(v[0] for v in acc.values()) or 1.0
ts = sum(v[1] for v in acc.values()) or 1.0
print(f"warp instructions {tot:.4g}, stall samples {ts:.4g}")
for k, v in sorted(acc.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0] / tot:6.3f} {v[1] / ts:6.3f} {k[0]}:{k[1]} {k[2]}")
print("SASS mix:", [(round(a, 3), b) for a, b in sorted(((v / tot, k) for k, v in sass.items()), reverse=True)[:20]])

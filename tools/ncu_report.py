"""Summarise an ncu report: per-launch key metrics, stall breakdown, SASS hotspots."""
import csv, subprocess, sys, io
rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
raw = page("raw")
h = raw[0]
want = ['launch__grid_size','gpu__time_duration.sum','smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct',
        'dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread']
idx = [h.index(w) for w in want if w in h]
print(' | '.join(h[i].split('__')[-1][:22] for i in idx))
for r in raw[2:]:
    print(r[h.index('Kernel Name')][:18], ' | '.join(r[i][:12] for i in idx))
stalls = [(i, n) for i, n in enumerate(h) if n.startswith('smsp__average_warp_latency_issue_stalled_') or n.startswith('smsp__pcsamp_warps_issue_stalled_')]
for r in raw[2:3]:
    tot = [(h[i].replace('smsp__pcsamp_warps_issue_stalled_',''), float(r[i] or 0)) for i, n in stalls if n.startswith('smsp__pcsamp') and not n.endswith('not_issued')]
    s = sum(v for _, v in tot) or 1
    print('stalls (launch 0):', ', '.join(f"{k}={v/s:.2f}" for k, v in sorted(tot, key=lambda x: -x[1])[:8]))
if len(sys.argv) > 2:
    k = int(sys.argv[2])
    src = page("source", ["--launch-skip", str(k), "--launch-count", "1"])
    his = [i for i, r in enumerate(src) if r and r[0] == 'Address']
    hh = src[his[0]]; data = [r for r in src[his[0]+1:(his[1]-1 if len(his) > 1 else None)] if len(r) == len(hh)]
    wi = hh.index('Warp Stall Sampling (All Samples)'); ei = hh.index('Instructions Executed'); si = hh.index('Source')
    f = lambda x: float(x) if x not in ('', '-') else 0.0
    tot = sum(f(r[wi]) for r in data)
    print('samples', tot)
    for r in sorted(data, key=lambda r: -f(r[wi]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
        print(r[0][-5:], f"{f(r[wi])/tot:.3f}", r[ei], r[si][:110])

#!/bin/bash
# Round-2 final state: full GPU suite, the default bench line, emulated 8-slab global mode, smoke()
mkdir -p gpurun_out/rec4
R=gpurun_out/rec4
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $R/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $R/pytest.log
timeout 600 python __graft_entry__.py smoke > $R/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $R/smoke.log
timeout 1500 python bench.py > $R/bench_c4.log 2>&1; echo "bench c4 rc=$?"; grep '^{' $R/bench_c4.log | tail -1 > $R/bench_c4.json
timeout 1500 python bench.py --mode global --emulate-ranks 8 --steps 5 --warmup 3 > $R/global8_c4.log 2>&1; echo "global8 rc=$?"; grep '^{' $R/global8_c4.log | tail -1 > $R/global8_c4.json
grep '^{' $R/bench_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("c4 ms/step %.2f value %.4g e2e %.4g lazy %.4g" % (d["ms_per_step"], d["value"], d["e2e"]["value"], d["e2e"]["lazy"]["value"]), d["roofline"]["breakdown_ms_per_step"], d["roofline"]["issue"])'
grep '^{' $R/global8_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print("global8 slowest %.2f" % e["slowest_rank_ms_per_step"], {k: round(v,2) for k,v in e["rank_ms_per_step"].items()})'

# A/B across configs + the bench: committed build (libtsb_old.so) vs working tree.
# usage: bash tools/gpu_ab_multi.sh "<configs comma list>" [pytest args...]
mkdir -p gpurun_out; rm -f gpurun_out/ab_multi.txt
cfgs=$1; shift
if [ $# -gt 0 ]; then timeout 900 python -m pytest "$@" -q -x 2>&1 | tail -5 > gpurun_out/ab_tests.txt; fi
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("bench", round(d["ms_per_step"],3), round(d["roofline"]["frac"],4))'
for i in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export TSB_LIB=$PWD/paper_1804_07250_b200/_lib/libtsb_old.so; else unset TSB_LIB; fi
    echo "== $v" >> gpurun_out/ab_multi.txt
    timeout 300 $B | python -c "$P" >> gpurun_out/ab_multi.txt 2>&1
    timeout 900 python tools/bench_configs.py --only $cfgs | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'][:50], {k: round(v,3) for k,v in d.items() if k in ('us_per_sweep','chain_sweeps_per_s','rotateable_fraction','us_per_sweep_all_chains','roofline_frac')})" >> gpurun_out/ab_multi.txt 2>&1
  done
done
unset TSB_LIB

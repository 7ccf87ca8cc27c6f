# A/B of an env setting on the working-tree build: "base" vs "$ENVSET" (e.g. TSB_DOM_WPL=3).
mkdir -p gpurun_out; rm -f gpurun_out/ab_env.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("bench", round(d["ms_per_step"],3), round(d["roofline"]["frac"],4))'
for i in 1 2; do
  for v in base env; do
    echo "== $v" >> gpurun_out/ab_env.txt
    if [ $v = env ]; then export $ENVSET; else unset ${ENVSET%%=*}; fi
    timeout 300 $B | python -c "$P" >> gpurun_out/ab_env.txt 2>&1
    timeout 900 python tools/bench_configs.py --only $CFGS | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'][:50], {k: round(v,3) for k,v in d.items() if k in ('us_per_sweep','chain_sweeps_per_s')})" >> gpurun_out/ab_env.txt 2>&1
  done
done

# Adaptive-order refresh interval (TSB_DOM_ORDER_EVERY) on the headline step.
mkdir -p gpurun_out; rm -f gpurun_out/order_every.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["warm"]["us_per_sweep"],3), round(d["collapsed"]["us_per_sweep"],4), round(d["collapsed"]["warm"]["us_per_sweep"],3))'
for rep in 1 2; do for e in 4 1 2 8 16; do
  echo "== every=$e $(TSB_DOM_ORDER_EVERY=$e timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/order_every.txt
done; done
echo "== adapt=0 $(TSB_DOM_ADAPT=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/order_every.txt

# With the hot-tile rule (libtsb_hot.so): adaptive-order refresh every 4 vs 8 vs 16 replays.
mkdir -p gpurun_out; rm -f gpurun_out/hot_every.txt
L=paper_1804_07250_b200/_lib
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["warm"]["us_per_sweep"],3), round(d["collapsed"]["us_per_sweep"],4), round(d["collapsed"]["warm"]["us_per_sweep"],3))'
for rep in 1 2 3; do for e in 4 8 16; do
  echo "== every=$e $(TSB_DOM_ORDER_EVERY=$e TSB_LIB=$PWD/$L/libtsb_hot.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/hot_every.txt
done; done
for e in 4 8; do echo "== every=$e C4 $(TSB_DOM_ORDER_EVERY=$e TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/$L/libtsb_hot.so timeout 600 python tools/bench_configs.py --only c4,strips | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/hot_every.txt; done

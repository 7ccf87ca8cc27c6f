# One replay-tail kernel (reorder + step advance + next colour table) instead
# of colors/order/advance kernels per 64-sweep replay (libtsb_tail.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/tail_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_tail.so timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/tail_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["collapsed"]["us_per_sweep"],4))'
for rep in 1 2 3; do for lib in libtsb.so libtsb_tail.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-warm | python -c "$P")" >> gpurun_out/tail_ab.txt
done; done
bash tools/ab_warm.sh $L/libtsb.so $L/libtsb_tail.so >> gpurun_out/tail_ab.txt 2>&1
for lib in libtsb.so libtsb_tail.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 900 python tools/bench_configs.py --only c1,c4,c5 | grep -o '"config": "[^"]\{0,12\}\|us_per_sweep": [0-9.]*\|chain_sweeps_per_s": [0-9.e+]*' | tr '\n' ' ')" >> gpurun_out/tail_ab.txt
done

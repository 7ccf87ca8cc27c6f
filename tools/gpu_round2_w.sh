# Persistent pipelined kernel with the adaptive tile order at Aztec 4096
# (TSB_DOM_PIPE=1 on libtsb_pa.so) vs the one-block-per-tile kernel.
mkdir -p gpurun_out; rm -f gpurun_out/pa_ab.txt
L=paper_1804_07250_b200/_lib
TSB_DOM_PIPE=1 TSB_LIB=$PWD/$L/libtsb_pa.so timeout 1500 python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py -q -x 2>&1 | tail -3 >> gpurun_out/pa_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["warm"]["us_per_sweep"],3), round(d["collapsed"]["us_per_sweep"],4), round(d["collapsed"]["warm"]["us_per_sweep"],3))'
for rep in 1 2; do
  echo "== base $(TSB_LIB=$PWD/$L/libtsb.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/pa_ab.txt
  echo "== pa   $(TSB_LIB=$PWD/$L/libtsb_pa.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/pa_ab.txt
  echo "== pa+pipe $(TSB_DOM_PIPE=1 TSB_LIB=$PWD/$L/libtsb_pa.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/pa_ab.txt
done

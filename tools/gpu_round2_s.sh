# A/B: three-IMAD 64-bit multiplies in mix64 (libtsb_mul3.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/mul3_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_mul3.so timeout 1200 python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py tests/test_sixvertex_gpu.py tests/test_lozenge_gpu.py -q -x 2>&1 | tail -3 >> gpurun_out/mul3_ab.txt
bash tools/ab_warm.sh $L/libtsb.so $L/libtsb_mul3.so $L/libtsb.so $L/libtsb_mul3.so >> gpurun_out/mul3_ab.txt 2>&1
for lib in libtsb.so libtsb_mul3.so libtsb.so libtsb_mul3.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 600 python tools/bench_configs.py --only c2,c3 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/mul3_ab.txt
  echo "== $lib plain $(TSB_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-collapsed | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["warm"]["us_per_sweep"])')" >> gpurun_out/mul3_ab.txt
done

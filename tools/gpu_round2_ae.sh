# p = 1/2 coins read off bit 63 of the draw (libtsb_half.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/half_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_half.so timeout 1800 python -m pytest tests/test_domino_gpu.py tests/test_lozenge_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py -k "not strips" -q -x 2>&1 | tail -3 >> gpurun_out/half_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["warm"]["us_per_sweep"],3), round(d["warm"]["roofline"]["frac"],4), round(d["collapsed"]["us_per_sweep"],4), round(d["collapsed"]["warm"]["us_per_sweep"],3))'
for rep in 1 2; do for lib in libtsb.so libtsb_half.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/half_ab.txt
done; done

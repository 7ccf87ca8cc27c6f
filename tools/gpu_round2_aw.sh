# warp_fire body inlined only into the lozenge and CFTP pair kernels (libtsb_inl2.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/inl2_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_inl2.so timeout 2400 python -m pytest tests/test_domino_gpu.py tests/test_lozenge_gpu.py tests/test_collapse_gpu.py -q -x 2>&1 | tail -2 >> gpurun_out/inl2_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["warm"]["us_per_sweep"],3), round(d["collapsed"]["us_per_sweep"],4), round(d["collapsed"]["warm"]["us_per_sweep"],3))'
for rep in 1 2; do for lib in libtsb.so libtsb_inl2.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/inl2_ab.txt
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib TSB_DOM_COLLAPSE=0 timeout 900 python tools/bench_configs.py --only c2,c4,c5 | grep -o 'us_per_sweep": [0-9.]*\|chain_sweeps_per_s": [0-9.e+]*' | tr '\n' ' ')" >> gpurun_out/inl2_ab.txt
done; done

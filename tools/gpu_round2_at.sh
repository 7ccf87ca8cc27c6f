# One-word domino tiles closed by the grid edge (libtsb_m1c.so) vs HEAD: tests and C5.
mkdir -p gpurun_out; rm -f gpurun_out/m1c_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_m1c.so timeout 2400 python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py tests/test_walk_subsets_gpu.py -k "not strips" -q -x 2>&1 | tail -3 >> gpurun_out/m1c_ab.txt
ls tests/*cftp* >> gpurun_out/m1c_ab.txt 2>&1
for rep in 1 2; do for lib in libtsb.so libtsb_m1c.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 900 python tools/bench_configs.py --only c1,c5 | grep -o 'us_per_sweep": [0-9.]*\|chain_sweeps_per_s": [0-9.e+]*' | tr '\n' ' ')" >> gpurun_out/m1c_ab.txt
done; done
for lib in libtsb.so libtsb_m1c.so; do
  echo "== $lib c5full8 $(TSB_C5_COUNT=8 TSB_LIB=$PWD/$L/$lib timeout 900 python tools/bench_configs.py --only c5full | grep -o '"seconds": [0-9.]*')" >> gpurun_out/m1c_ab.txt
done

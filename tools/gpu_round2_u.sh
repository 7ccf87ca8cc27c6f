# Pipelined C4 kernel: launch sweeps resolved once per block and tile
# coordinates prefetched two tiles ahead (libtsb_pf.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/pf_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_pf.so timeout 1500 python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py -k "domino or c4 or metric or collapse" -q -x 2>&1 | tail -3 >> gpurun_out/pf_ab.txt
for rep in 1 2; do for lib in libtsb.so libtsb_pf.so; do
  for col in 0 1; do
    echo "== $lib collapse=$col c4 $(TSB_DOM_COLLAPSE=$col TSB_LIB=$PWD/$L/$lib timeout 600 python tools/bench_configs.py --only c4 | grep -o 'us_per_sweep": [0-9.]*')" >> gpurun_out/pf_ab.txt
  done
done; done
bash tools/ab_warm.sh $L/libtsb.so $L/libtsb_pf.so >> gpurun_out/pf_ab.txt 2>&1

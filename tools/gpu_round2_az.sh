# Lozenge: class masks by shift (libtsb_m3.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/m3_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_m3.so timeout 1800 python -m pytest tests/test_lozenge_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py tests/test_observables_gpu.py -k "lozenge or loz or c2" -q -x 2>&1 | tail -3 >> gpurun_out/m3_ab.txt
for rep in 1 2; do for lib in libtsb.so libtsb_m3.so; do for col in 0 1; do
  echo "== $lib collapse=$col $(TSB_LZ_COLLAPSE=$col TSB_LIB=$PWD/$L/$lib timeout 600 python tools/bench_configs.py --only c2,batched | grep -o 'us_per_sweep": [0-9.]*\|attempts_per_s": [0-9.e+]*' | tr '\n' ' ')" >> gpurun_out/m3_ab.txt
done; done; done

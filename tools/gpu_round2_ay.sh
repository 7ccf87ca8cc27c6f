# Lozenge: 22-row tiles (one block per SM) for single lattices whose 16-row
# tiles spill past one block per SM (libtsb_l22.so; TSB_LZ_TALL=0 off) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/l22_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_l22.so timeout 1800 python -m pytest tests/test_lozenge_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py tests/test_observables_gpu.py tests/test_heights_gpu.py -k "lozenge or loz or c2" -q -x 2>&1 | tail -3 >> gpurun_out/l22_ab.txt
for rep in 1 2; do for v in "libtsb.so -1" "libtsb_l22.so -1" "libtsb_l22.so 0"; do set -- $v; for col in 0 1; do
  echo "== $1 tall=$2 collapse=$col $(TSB_LZ_TALL=$2 TSB_LZ_COLLAPSE=$col TSB_LIB=$PWD/$L/$1 timeout 600 python tools/bench_configs.py --only c2 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/l22_ab.txt
done; done; done

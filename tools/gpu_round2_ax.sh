# Six-vertex: block barrier only before a sweep of the other row parity (libtsb_svb.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/svb_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_svb.so timeout 1800 python -m pytest tests/test_sixvertex_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py tests/test_oracle_golden.py -k "sixvertex or c3 or sv" -q -x 2>&1 | tail -3 >> gpurun_out/svb_ab.txt
for rep in 1 2; do for v in "libtsb.so 1" "libtsb_svb.so 1"; do set -- $v; for col in 0 1; do
  echo "== $1 xw=$2 collapse=$col $(TSB_SV_XW=$2 TSB_SV_COLLAPSE=$col TSB_LIB=$PWD/$L/$1 timeout 600 python tools/bench_configs.py --only c3 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/svb_ab.txt
done; done; done

# Six-vertex: kind and diagonal masks only in warps with candidates (libtsb_svl.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/svl_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_svl.so timeout 1800 python -m pytest tests/test_sixvertex_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py -k "sixvertex or c3" -q -x 2>&1 | tail -3 >> gpurun_out/svl_ab.txt
for rep in 1 2; do for lib in libtsb.so libtsb_svl.so; do for col in 0 1; do
  echo "== $lib collapse=$col $(TSB_SV_COLLAPSE=$col TSB_LIB=$PWD/$L/$lib timeout 600 python tools/bench_configs.py --only c3 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/svl_ab.txt
done; done; done

# Lozenge 32-row / K = 8 tiles for single lattices (libtsb_lz32.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/lz32_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_lz32.so timeout 1500 python -m pytest tests/test_lozenge_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py -k "lozenge or loz or c2" -q -x 2>&1 | tail -3 >> gpurun_out/lz32_ab.txt
for rep in 1 2; do for lib in libtsb.so libtsb_lz32.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 600 python tools/bench_configs.py --only c2 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/lz32_ab.txt
done; done
for k in 4 16; do echo "== lz32 K=$k $(TSB_LZ_K=$k TSB_LIB=$PWD/$L/libtsb_lz32.so timeout 600 python tools/bench_configs.py --only c2 | grep -o 'us_per_sweep": [0-9.]*')" >> gpurun_out/lz32_ab.txt; done
TSB_LIB=$PWD/$L/libtsb_lz32.so timeout 900 ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats -k regex:lz_multi -s 40 -c 1 python tools/bench_configs.py --only c2 > gpurun_out/lz32_ncu.txt 2>&1

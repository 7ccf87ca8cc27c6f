mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sixvertex_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/sv_tests.txt
rm -f gpurun_out/sv_tune.txt
for cfg in "8 16 0" "8 16 1" "8 16 2" "4 16 1" "4 8 1" "8 16 3"; do set -- $cfg; echo "K=$1 NW=$2 WPL=$3" >> gpurun_out/sv_tune.txt; TSB_SV_K=$1 TSB_SV_NW=$2 TSB_SV_WPL=$3 timeout 300 python tools/bench_configs.py --only c3 >> gpurun_out/sv_tune.txt 2>&1; done

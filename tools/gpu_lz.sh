mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lozenge_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/lz_tests.txt
rm -f gpurun_out/lz_tune.txt
for k in 2 4 8; do echo "K=$k" >> gpurun_out/lz_tune.txt; TSB_LZ_K=$k timeout 300 python tools/bench_configs.py --only c2 >> gpurun_out/lz_tune.txt 2>&1; done

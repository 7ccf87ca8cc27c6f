python -m pytest tests -m gpu -x -q -k "not c2_ and not c3_" 2>&1 | tail -5 > gpurun_out/r2_g_tests.log
for c in 0 1; do echo "collapse=$c $(TSB_DOM_COLLAPSE=$c python tools/time_warm.py 2>&1 | tail -1)"; done > gpurun_out/r2_g_timing.txt
echo "C4 collapse=1 $(timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1)" >> gpurun_out/r2_g_timing.txt
echo "C5 $(timeout 900 python tools/bench_configs.py --only c5 2>&1 | tail -1)" >> gpurun_out/r2_g_timing.txt
cat gpurun_out/r2_g_tests.log gpurun_out/r2_g_timing.txt

python -m pytest tests -m gpu -x -q -k "not c2 and not c3_" 2>&1 | tail -3 > gpurun_out/r2_t9_collapse_on.log
TSB_DOM_COLLAPSE=0 python -m pytest tests/test_domino_gpu.py tests/test_walk_host_gpu.py tests/test_strips_gpu.py tests/test_configs_gpu.py -x -q -k "not c2 and not c3_" 2>&1 | tail -3 > gpurun_out/r2_t9_collapse_off.log
for c in 0 1; do echo "collapse=$c $(TSB_DOM_COLLAPSE=$c python tools/time_warm.py 2>&1 | tail -1)"; done > gpurun_out/r2_t9_timing.txt
cat gpurun_out/r2_t9_collapse_on.log gpurun_out/r2_t9_collapse_off.log gpurun_out/r2_t9_timing.txt

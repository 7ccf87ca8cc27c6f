rm -f gpurun_out/r2_i.txt
for rep in 1 2; do for lib in libtsb_r1.so libtsb_763f3a2.so libtsb.so; do
  echo "== $lib c4 $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1 | grep -o '"us_per_sweep": [0-9.]*')" >> gpurun_out/r2_i.txt
done; done
for lib in libtsb_r1.so libtsb.so; do
  echo "== $lib $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/time_warm.py 2>&1 | tail -1)" >> gpurun_out/r2_i.txt
done
echo "== libtsb.so collapse=1 $(python tools/time_warm.py 2>&1 | tail -1)" >> gpurun_out/r2_i.txt
python -m pytest tests/test_collapse_gpu.py tests/test_domino_gpu.py tests/test_configs_gpu.py -q -x -k "not c2_ and not c3_" 2>&1 | tail -2 >> gpurun_out/r2_i.txt
cat gpurun_out/r2_i.txt

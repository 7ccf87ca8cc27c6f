mkdir -p gpurun_out; rm -f gpurun_out/lz_knobs.txt
timeout 600 python -m pytest tests/test_lozenge_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/lz_knob_tests.txt
for v in old new; do for k in 4 8; do
  if [ $v = old ]; then export TSB_LIB=$PWD/paper_1804_07250_b200/_lib/libtsb_old.so; else unset TSB_LIB; fi
  echo "$v K=$k" >> gpurun_out/lz_knobs.txt
  TSB_LZ_K=$k timeout 300 python tools/bench_configs.py --only c2 | grep -o 'us_per_sweep": [0-9.]*' >> gpurun_out/lz_knobs.txt
done; done

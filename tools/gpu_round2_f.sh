rm -f gpurun_out/r2_f.txt
for rep in 1 2; do for lib in libtsb_r1.so libtsb.so; do
  echo "== $lib $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1 | grep -o '"us_per_sweep": [0-9.]*')" >> gpurun_out/r2_f.txt
done; done
cat gpurun_out/r2_f.txt

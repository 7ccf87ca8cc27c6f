rm -f gpurun_out/r2_h.txt
for rep in 1 2; do for lib in libtsb_r1.so libtsb_763f3a2.so libtsb_3a0f3e8.so libtsb_71daf17.so libtsb.so; do
  echo "== $lib $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1 | grep -o '"us_per_sweep": [0-9.]*')" >> gpurun_out/r2_h.txt
done; done
cat gpurun_out/r2_h.txt

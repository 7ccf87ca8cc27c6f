# A/B: round-1 final build vs current (2-stage HEAD build) vs 3-stage, C4 and Aztec 4096
rm -f gpurun_out/r2_e.txt
for rep in 1 2; do
for lib in libtsb_r1.so libtsb_p2.so libtsb.so; do
  echo "== $lib $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1 | grep -o '"us_per_sweep": [0-9.]*')" >> gpurun_out/r2_e.txt
done; done
for lib in libtsb_r1.so libtsb_p2.so libtsb.so; do
  echo "== $lib $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/time_warm.py 2>&1 | tail -1)" >> gpurun_out/r2_e.txt
done
cat gpurun_out/r2_e.txt

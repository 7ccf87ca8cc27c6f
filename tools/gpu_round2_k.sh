for rep in 1 2; do for lib in libtsb_r1.so libtsb_nomask.so libtsb.so; do
  echo "== $lib c4 $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1 | grep -o '"us_per_sweep": [0-9.]*')"
done; done
for lib in libtsb_nomask.so libtsb.so; do
  echo "== $lib $(TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/time_warm.py 2>&1 | tail -1)"
done
python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py -q -x 2>&1 | tail -2

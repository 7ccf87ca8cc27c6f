for rep in 1 2; do for lib in libtsb_head.so libtsb_sw2.so; do
  for c in 0 1; do echo "== $lib collapse=$c $(TSB_DOM_COLLAPSE=$c TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/time_warm.py 2>&1 | tail -1)"; done
done; done
python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py -q -x -k "not c2_ and not c3_" 2>&1 | tail -2

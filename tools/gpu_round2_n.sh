for rep in 1 2; do for lib in libtsb_sw2.so libtsb_svpad.so libtsb_svquad.so; do
  echo "== $lib $(TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/bench_configs.py --only c3 2>&1 | grep -o '"us_per_sweep": [0-9.]*' | tr '\n' ' ') plain: $(TSB_SV_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/bench_configs.py --only c3 2>&1 | grep -o '"us_per_sweep": [0-9.]*' | tr '\n' ' ')"
done; done
python -m pytest tests/test_sixvertex_gpu.py tests/test_collapse_gpu.py -q -x 2>&1 | tail -2
TSB_LIB=$PWD/paper_1804_07250_b200/_lib/libtsb_svquad.so python -m pytest tests/test_sixvertex_gpu.py -q -x 2>&1 | tail -2

for rep in 1 2; do for lib in libtsb_sw2.so libtsb_q4.so; do
  for c in 0 1; do echo "== $lib collapse=$c $(TSB_DOM_COLLAPSE=$c TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/time_warm.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["warm"]["us_per_sweep"],3), round(d["tmax"]["us_per_sweep"],3))')"; done
done; done
python tools/bench_configs.py --only c2,c3 2>&1 | grep -o '"us_per_sweep": [0-9.]*' | tr '\n' ' '
python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py tests/test_lozenge_gpu.py tests/test_sixvertex_gpu.py -q -x 2>&1 | tail -2

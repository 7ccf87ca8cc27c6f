for rep in 1 2; do for lib in libtsb_sw2.so libtsb_v_cmp.so libtsb_v_qs.so libtsb_v_bal.so libtsb_v_both.so; do
  r=""
  for c in 0 1; do r="$r $(TSB_DOM_COLLAPSE=$c TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/time_warm.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["warm"]["us_per_sweep"],3), round(d["tmax"]["us_per_sweep"],3))')"; done
  echo "== $lib warm/tmax plain, collapsed: $r c2: $(TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib python tools/bench_configs.py --only c2 2>&1 | grep -o '"us_per_sweep": [0-9.]*')"
done; done

# Tile costs recorded only in the replays that reorder (libtsb_meas.so) vs HEAD.
mkdir -p gpurun_out; rm -f gpurun_out/meas_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_meas.so timeout 1800 python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py tests/test_configs_gpu.py tests/test_strips_gpu.py -q -x 2>&1 | tail -2 >> gpurun_out/meas_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), round(d["warm"]["us_per_sweep"],3), round(d["collapsed"]["us_per_sweep"],4), round(d["collapsed"]["warm"]["us_per_sweep"],3))'
for rep in 1 2; do for lib in libtsb.so libtsb_meas.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "$P")" >> gpurun_out/meas_ab.txt
done; done

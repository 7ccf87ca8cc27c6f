mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_domino_gpu.py tests/test_strips_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/dom_tests.txt
rm -f gpurun_out/dom_tune.txt
for cfg in "1 2" "1 4" "2 2" "2 4"; do set -- $cfg; echo "RPW=$1 K=$2" >> gpurun_out/dom_tune.txt; TSB_DOM_RPW=$1 TSB_DOM_K=$2 TSB_DOM_FLAGS=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/dom_tune.txt 2>&1; done

# Refresh of the lozenge numbers after the class-mask change.
set -x; O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests/test_lozenge_gpu.py tests/test_configs_gpu.py tests/test_collapse_gpu.py -k "lozenge or loz or c2" -q 2>&1 | tail -2 > $O/pytest_lz.txt
TSB_DOM_COLLAPSE=0 TSB_SV_COLLAPSE=0 TSB_LZ_COLLAPSE=0 timeout 900 python tools/bench_configs.py --only c2,batched > $O/lz_plain.jsonl 2>&1
timeout 900 python tools/bench_configs.py --only c2,batched > $O/lz_collapsed.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lz_multi -s 200 -c 1 -o $O/prof_lz python tools/prof_driver.py lz > /dev/null 2>&1
python tools/ncu_summary.py $O/prof_lz.ncu-rep --sass 25 > $O/prof_lz_ncu.txt 2>&1

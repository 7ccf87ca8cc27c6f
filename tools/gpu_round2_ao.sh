# Refresh of the six-vertex numbers after the candidate-test change.
set -x; O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests/test_sixvertex_gpu.py tests/test_configs_gpu.py tests/test_collapse_gpu.py tests/test_observables_gpu.py tests/test_archive_gpu.py -k "sixvertex or c3 or sv" -q 2>&1 | tail -2 > $O/pytest_sv.txt
TSB_DOM_COLLAPSE=0 TSB_SV_COLLAPSE=0 TSB_LZ_COLLAPSE=0 timeout 900 python tools/bench_configs.py --only c3,batched > $O/sv_plain.jsonl 2>&1
timeout 900 python tools/bench_configs.py --only c3,batched > $O/sv_collapsed.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_multi -s 200 -c 1 -o $O/prof_sv python tools/prof_driver.py sv > /dev/null 2>&1
python tools/ncu_summary.py $O/prof_sv.ncu-rep --sass 25 > $O/prof_sv_ncu.txt 2>&1

# Bench line and warm ncu captures from the 4 n^2 warm state.
set -x; O=gpurun_out/final; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
TSB_DOM_COLLAPSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_multi -s 100 -c 1 -o $O/prof_multi_warm python tools/prof_driver.py dom --state bench_data/aztec4096_warm.npz --warm 256 --sweeps 64 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_multi -s 60 -c 1 -o $O/prof_multi_warm_collapsed python tools/prof_driver.py dom --state bench_data/aztec4096_warm.npz --warm 512 --sweeps 64 > /dev/null 2>&1
for r in prof_multi_warm prof_multi_warm_collapsed; do python tools/ncu_summary.py $O/$r.ncu-rep --sass 25 > $O/${r}_ncu.txt 2>&1; done
TSB_DOM_COLLAPSE=0 timeout 600 python tools/bench_configs.py --only mixed > $O/mixed_plain.jsonl 2>&1

# Round-2 final measurements on one B200 -> gpurun_out/final/ (copied to profiles/round2_*)
set -x; O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt; nproc >> $O/gpu.txt; lscpu | grep "Model name" >> $O/gpu.txt
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15 > $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-warm --no-collapsed > $O/bench_2ranks.json 2> $O/bench_2ranks.err
TSB_DOM_COLLAPSE=0 TSB_SV_COLLAPSE=0 TSB_LZ_COLLAPSE=0 timeout 1500 python tools/bench_configs.py --only c1,c2,c3,c4,c5,batched,strips > $O/configs_plain.jsonl 2>&1
timeout 1500 python tools/bench_configs.py --only c1,c2,c3,c4,c5,batched,strips > $O/configs_collapsed.jsonl 2>&1
TSB_C5_COUNT=8 timeout 900 python tools/bench_configs.py --only c5full > $O/c5full8.jsonl 2>&1
TSB_C5_COUNT=64 timeout 1500 python tools/bench_configs.py --only c5full > $O/c5full64.jsonl 2>&1
python tools/time_heights.py > $O/heights.jsonl 2>&1
ARGS="--order 4096 --steps 2 --warmup 1 --sweeps-per-step 128 --no-e2e --no-cpu-baseline --no-warm --no-collapsed"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 150 --csv --log-file $O/launches_4096.csv python bench.py $ARGS > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_multi -s 100 -c 2 -o $O/prof_multi python bench.py $ARGS > /dev/null 2>&1
TSB_DOM_COLLAPSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_multi -s 100 -c 1 -o $O/prof_multi_warm python tools/prof_driver.py dom --state bench_data/aztec4096_warm.npz --warm 256 --sweeps 64 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_multi -s 60 -c 1 -o $O/prof_multi_warm_collapsed python tools/prof_driver.py dom --state bench_data/aztec4096_warm.npz --warm 512 --sweeps 64 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_multi -s 200 -c 1 -o $O/prof_sv python tools/prof_driver.py sv > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lz_multi -s 200 -c 1 -o $O/prof_lz python tools/prof_driver.py lz > /dev/null 2>&1
TSB_DOM_COLLAPSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_multi_pipe -s 20 -c 1 -o $O/prof_pipe python tools/prof_driver.py dom --n 16384 --warm 64 --sweeps 32 > /dev/null 2>&1
for r in prof_multi prof_multi_warm prof_multi_warm_collapsed prof_sv prof_lz prof_pipe; do python tools/ncu_summary.py $O/$r.ncu-rep --sass 25 > $O/${r}_ncu.txt 2>&1; done
bash tools/sanitize.sh > /dev/null 2>&1; cp gpurun_out/sanitizer.txt $O/sanitizer.txt
rm -f gpurun_out/san_*.log
ls -la $O

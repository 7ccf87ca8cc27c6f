# Full round check on one B200: GPU tests, smoke, bench (both arms), configs, ncu.
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"; free -g | head -2
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.txt 2>&1
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.txt 2>&1
ARGS="--order 4096 --steps 2 --warmup 1 --sweeps-per-step 128 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --cache-control none -s 200 -c 200 --csv --log-file gpurun_out/launches_4096.csv python bench.py $ARGS > gpurun_out/prof_launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:domino_multi -s 100 -c 2 -o gpurun_out/prof_multi_warm python bench.py $ARGS > gpurun_out/prof_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:sv_multi -s 200 -c 1 -o gpurun_out/prof_sv_warm python tools/prof_driver.py sv > gpurun_out/prof_sv.txt 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:lz_multi -s 200 -c 1 -o gpurun_out/prof_lz_warm python tools/prof_driver.py lz > gpurun_out/prof_lz.txt 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:domino_multi_pipe -s 20 -c 1 -o gpurun_out/prof_multi_pipe python tools/dbg_sizes.py 16384 > gpurun_out/prof_multi_pipe.txt 2>&1
timeout 1200 python tools/bench_configs.py --only strips,batched > gpurun_out/configs_extra.txt 2>&1

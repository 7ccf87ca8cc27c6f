set -x; mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py > gpurun_out/configs.txt 2>&1
ARGS="--order 4096 --steps 2 --warmup 1 --sweeps-per-step 128 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --cache-control none -s 600 -c 300 --csv --log-file gpurun_out/launches_4096.csv python bench.py $ARGS > gpurun_out/prof_bench_4096.txt 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:domino_sweep -s 300 -c 2 -o gpurun_out/prof_sweep python bench.py $ARGS > gpurun_out/prof_full.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1

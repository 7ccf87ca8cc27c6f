set -x; mkdir -p gpurun_out
for O in 512 4096; do
ARGS="--order $O --steps 2 --warmup 1 --sweeps-per-step 64 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/launches_$O.csv python bench.py $ARGS > gpurun_out/prof_bench_$O.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:domino_sweep -s 200 -c 2 -o gpurun_out/prof_sweep python bench.py --order 4096 --steps 2 --warmup 1 --sweeps-per-step 128 --no-e2e --no-cpu-baseline > gpurun_out/prof_full.txt 2>&1

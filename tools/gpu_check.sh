set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 300 python bench.py --order 512 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench512.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.txt 2>&1
nproc; lscpu | grep "Model name"

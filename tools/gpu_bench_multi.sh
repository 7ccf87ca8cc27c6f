# N>1 bench paths on ONE GPU (processes share cuda:0; numbers are not scaling
# measurements, only a check that the torchrun paths run end to end).
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for mode in "" "--replicas"; do
  echo "== world 2 $mode" >> gpurun_out/bench_multi.txt
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/bench_shared_gpu.py --gpus 2 --steps 3 --warmup 3 --order 1024 --sweeps-per-step 256 --no-cpu-baseline $mode >> gpurun_out/bench_multi.txt 2>&1
done

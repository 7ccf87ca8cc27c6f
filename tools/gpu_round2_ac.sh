# Extend the committed warm state from 2^24 to 2^26 sweeps (4 n^2), then time it.
mkdir -p gpurun_out/warm
cp bench_data/aztec4096_warm.npz gpurun_out/warm/old.npz
timeout 2400 python tools/make_warm_state.py gpurun_out/warm/aztec4096_warm.npz --from gpurun_out/warm/old.npz > gpurun_out/warm/trace.jsonl 2>&1
cp gpurun_out/warm/aztec4096_warm.npz bench_data/aztec4096_warm.npz
timeout 600 python tools/time_warm.py > gpurun_out/warm/time_warm.json 2>&1

# A/B: block-pooled coins (TSB_POOL=1 build) vs the per-warp coin queues.
mkdir -p gpurun_out; rm -f gpurun_out/pool_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_pool.so timeout 900 python -m pytest tests/test_domino_gpu.py tests/test_collapse_gpu.py -q -x 2>&1 | tail -3 >> gpurun_out/pool_ab.txt
bash tools/ab_warm.sh $L/libtsb.so $L/libtsb_pool.so $L/libtsb.so $L/libtsb_pool.so >> gpurun_out/pool_ab.txt 2>&1
for lib in libtsb.so libtsb_pool.so; do
  echo "== $lib c4 $(TSB_LIB=$PWD/$L/$lib timeout 600 python tools/bench_configs.py --only c4 | grep -o 'us_per_sweep": [0-9.]*')" >> gpurun_out/pool_ab.txt
done

# A/B on a config bench: alternate the committed build (libtsb_old.so) and the working tree.
# usage: bash tools/gpu_ab_cfg.sh <config> [extra pytest targets]
mkdir -p gpurun_out; rm -f gpurun_out/ab_cfg.txt
cfg=$1; shift
if [ $# -gt 0 ]; then timeout 900 python -m pytest "$@" -q -x 2>&1 | tail -5 > gpurun_out/ab_tests.txt; fi
for i in 1 2; do
  echo "old:" >> gpurun_out/ab_cfg.txt; TSB_LIB=$PWD/paper_1804_07250_b200/_lib/libtsb_old.so timeout 600 python tools/bench_configs.py --only $cfg >> gpurun_out/ab_cfg.txt 2>&1
  echo "new:" >> gpurun_out/ab_cfg.txt; timeout 600 python tools/bench_configs.py --only $cfg >> gpurun_out/ab_cfg.txt 2>&1
done

# C3 single-chain tile-shape sweep (K sweeps per launch, NW warps per block,
# WPL words per lane; default = auto) on the HEAD build.
mkdir -p gpurun_out; rm -f gpurun_out/sv_shapes.txt
for cfg in "def def def" "8 15 1" "8 16 1" "4 16 1" "4 8 1" "8 15 2" "8 16 2" "4 8 2" "16 16 1" "4 15 1"; do
  set -- $cfg
  unset TSB_SV_K TSB_SV_NW TSB_SV_WPL
  [ $1 != def ] && export TSB_SV_K=$1 TSB_SV_NW=$2 TSB_SV_WPL=$3
  echo "K=$1 NW=$2 WPL=$3 $(timeout 300 python tools/bench_configs.py --only c3 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/sv_shapes.txt
done

# C3 tile shapes with the east-boundary-word tiles (K sweeps per launch, NW warps).
mkdir -p gpurun_out; rm -f gpurun_out/sv_shapes_xw.txt
for cfg in "def def" "8 15" "8 16" "4 8" "4 15" "4 16"; do
  set -- $cfg
  unset TSB_SV_K TSB_SV_NW
  [ $1 != def ] && export TSB_SV_K=$1 TSB_SV_NW=$2
  echo "K=$1 NW=$2 $(timeout 300 python tools/bench_configs.py --only c3 | grep -o 'us_per_sweep": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/sv_shapes_xw.txt
done

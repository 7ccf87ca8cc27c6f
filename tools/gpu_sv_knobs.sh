mkdir -p gpurun_out; rm -f gpurun_out/sv_knobs.txt
for cfg in "0 4" "1 4" "0 0" "1 0" "0 1000" "1 1000"; do set -- $cfg
  echo "NO_RBOUND=$1 SPARSE=$2" >> gpurun_out/sv_knobs.txt
  if [ $1 = 1 ]; then export TSB_SV_NO_RBOUND=1; else unset TSB_SV_NO_RBOUND; fi
  TSB_SV_SPARSE=$2 timeout 300 python tools/bench_configs.py --only c3 | grep -o 'Delta=[^ ]*\|us_per_sweep": [0-9.]*' | paste - - >> gpurun_out/sv_knobs.txt
done

# round 2: full GPU suite (collapsing on), the collapse tests, C2/C3 knob A/B
python -m pytest tests -m gpu -x -q -k "not c2_ and not c3_" 2>&1 | tail -3 > gpurun_out/r2_c_tests.log
rm -f gpurun_out/r2_c_cfg.txt
for cfg in "SV=1 LZ=1 NW=16" "SV=0 LZ=0 NW=16" "SV=1 LZ=1 NW=15"; do
  set -- $cfg; sv=${1#SV=}; lz=${2#LZ=}; nw=${3#NW=}
  echo "== $cfg" >> gpurun_out/r2_c_cfg.txt
  TSB_SV_COLLAPSE=$sv TSB_LZ_COLLAPSE=$lz TSB_SV_NW=$nw timeout 600 python tools/bench_configs.py --only c2,c3 2>&1 | grep -o '"config": "[^"]*"\|"us_per_sweep": [0-9.]*' | paste - - >> gpurun_out/r2_c_cfg.txt
done
cat gpurun_out/r2_c_tests.log gpurun_out/r2_c_cfg.txt

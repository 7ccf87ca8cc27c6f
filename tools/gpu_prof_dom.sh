mkdir -p gpurun_out
for cfg in "1 2 0" "2 4 0"; do set -- $cfg
TSB_DOM_RPW=$1 TSB_DOM_K=$2 TSB_DOM_FLAGS=$3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:domino_tb -s 60 -c 1 -o gpurun_out/prof_dom_$1_$2_$3 python tools/prof_driver.py dom --warm 256 --sweeps 64 > gpurun_out/prof_dom_$1_$2.txt 2>&1
done

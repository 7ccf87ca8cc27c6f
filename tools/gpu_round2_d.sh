# C4 pipe depth A/B, sv/lz ncu captures
rm -f gpurun_out/r2_d_c4.txt
for lib in libtsb_p2.so libtsb.so; do
  echo "== $lib" >> gpurun_out/r2_d_c4.txt
  TSB_DOM_COLLAPSE=0 TSB_LIB=$PWD/paper_1804_07250_b200/_lib/$lib timeout 600 python tools/bench_configs.py --only c4 2>&1 | tail -1 >> gpurun_out/r2_d_c4.txt
done
ncu --set full --clock-control none --import-source on -k regex:domino_multi_pipe -s 20 -c 1 -o gpurun_out/r2_pipe3 python tools/prof_driver.py dom --n 16384 --warm 64 --sweeps 32 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2_pipe3.ncu-rep --sass 0 > gpurun_out/r2_pipe3_ncu.txt 2>&1
TSB_SV_NW=15 ncu --set full --clock-control none --import-source on -k regex:sv_multi -s 200 -c 1 -o gpurun_out/r2_sv python tools/prof_driver.py sv > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2_sv.ncu-rep --sass 30 > gpurun_out/r2_sv_ncu.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:lz_multi -s 200 -c 1 -o gpurun_out/r2_lz python tools/prof_driver.py lz > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2_lz.ncu-rep --sass 30 > gpurun_out/r2_lz_ncu.txt 2>&1
cat gpurun_out/r2_d_c4.txt; head -30 gpurun_out/r2_pipe3_ncu.txt; head -32 gpurun_out/r2_sv_ncu.txt; head -32 gpurun_out/r2_lz_ncu.txt

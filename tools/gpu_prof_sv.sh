mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sv_multi -s 200 -c 2 -o gpurun_out/prof_sv python tools/prof_driver.py sv > gpurun_out/prof_sv.txt 2>&1

# A/B of the window latency probe: committed build vs working tree.
mkdir -p gpurun_out; rm -f gpurun_out/ab_window.txt
for v in old new; do
  if [ $v = old ]; then export TSB_LIB=$PWD/paper_1804_07250_b200/_lib/libtsb_old.so; else unset TSB_LIB; fi
  echo "== $v" >> gpurun_out/ab_window.txt
  timeout 300 python tools/dbg_window.py >> gpurun_out/ab_window.txt 2>&1
done

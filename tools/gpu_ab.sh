# A/B: alternate the committed build (TSB_LIB=libtsb_old.so) and the working tree build.
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["frac"],4))'
for i in 1 2 3; do
  echo -n "old: " >> gpurun_out/ab.txt; TSB_LIB=$PWD/paper_1804_07250_b200/_lib/libtsb_old.so timeout 300 $B | python -c "$P" >> gpurun_out/ab.txt 2>&1
  echo -n "new: " >> gpurun_out/ab.txt; TSB_DOM_RPW=1 TSB_DOM_K=2 timeout 300 $B | python -c "$P" >> gpurun_out/ab.txt 2>&1
done

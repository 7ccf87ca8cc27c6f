# Host copy threads (TSB_COPY_THREADS) vs staged copy times and e2e.
mkdir -p gpurun_out; rm -f gpurun_out/threads_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["e2e"]["value"]/1e12,4), round(d["e2e"]["collapsed_library_default"]/1e12,4))'
for th in 4 8 12 16; do
  echo "== threads=$th $(TSB_COPY_THREADS=$th timeout 300 python tools/probe_host_copies.py | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: round(v,3) for k,v in d.items() if k.endswith("_ms")})')" >> gpurun_out/threads_ab.txt
  echo "== threads=$th e2e $(TSB_COPY_THREADS=$th timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-warm --no-collapsed | python -c "$P")" >> gpurun_out/threads_ab.txt
done

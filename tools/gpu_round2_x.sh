# Nibble-staged domino uploads / downloads (libtsb_nib.so) vs HEAD: tests and e2e.
mkdir -p gpurun_out; rm -f gpurun_out/nib_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_nib.so timeout 1800 python -m pytest tests/test_domino_gpu.py tests/test_walk_host_gpu.py tests/test_collapse_gpu.py tests/test_strips_gpu.py tests/test_configs_gpu.py -k "not c4_aztec_16384_strips and not memory_sharded" -q -x 2>&1 | tail -3 >> gpurun_out/nib_ab.txt
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["e2e"]["value"]/1e12,4), round(d["e2e"]["collapsed_library_default"]/1e12,4), d["e2e"]["h2d_bytes_per_step"])'
for rep in 1 2; do for lib in libtsb.so libtsb_nib.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-warm --no-collapsed | python -c "$P")" >> gpurun_out/nib_ab.txt
done; done
for lib in libtsb.so libtsb_nib.so; do
  echo "== $lib probe" >> gpurun_out/nib_ab.txt
  TSB_LIB=$PWD/$L/$lib timeout 300 python tools/probe_host_copies.py >> gpurun_out/nib_ab.txt 2>&1
done

# Height export through pinned staging (libtsb_hd.so) vs the pageable cudaMemcpy (HEAD).
mkdir -p gpurun_out; rm -f gpurun_out/hd_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_hd.so timeout 1800 python -m pytest tests/test_heights_gpu.py tests/test_domino_gpu.py tests/test_lozenge_gpu.py tests/test_configs_gpu.py -k "height or extremal or c2 or metric or golden" -q -x 2>&1 | tail -2 >> gpurun_out/hd_ab.txt
for lib in libtsb.so libtsb_hd.so libtsb.so libtsb_hd.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 600 python tools/time_heights.py 2>&1 | grep -o '"order": [0-9]*\|"path": "[a-z-]*"\|"heights_ms": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/hd_ab.txt
done

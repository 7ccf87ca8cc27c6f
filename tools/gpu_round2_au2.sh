# Four-agreeing-bits rotateable test in every domino kernel (libtsb_d4.so): full GPU suite, C1, C5.
mkdir -p gpurun_out; rm -f gpurun_out/d4b_ab.txt
L=paper_1804_07250_b200/_lib
TSB_LIB=$PWD/$L/libtsb_d4.so timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/d4b_ab.txt
for rep in 1 2; do for lib in libtsb.so libtsb_d4.so; do
  echo "== $lib $(TSB_LIB=$PWD/$L/$lib timeout 900 python tools/bench_configs.py --only c1,c5 | grep -o 'us_per_sweep": [0-9.]*\|chain_sweeps_per_s": [0-9.e+]*' | tr '\n' ' ')" >> gpurun_out/d4b_ab.txt
done; done
for lib in libtsb.so libtsb_d4.so; do
  echo "== $lib c5full8 $(TSB_C5_COUNT=8 TSB_LIB=$PWD/$L/$lib timeout 900 python tools/bench_configs.py --only c5full | grep -o '"seconds": [0-9.]*')" >> gpurun_out/d4b_ab.txt
done

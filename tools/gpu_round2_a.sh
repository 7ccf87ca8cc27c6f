set -x
python -c "
import time, paper_1804_07250_b200 as ts
d=ts.TriDomain.hexagon(1000,1000,1000); ts.loz_extremal(ts.TriDomain.hexagon(10,10,10))
t=time.time(); ts.loz_extremal(d); print('loz_extremal 1000', time.time()-t)
d=ts.Domain.aztec(1024); t=time.time(); ts.extremal_tilings(d); print('domino extremal aztec 1024', time.time()-t)
d=ts.Domain.rectangle(1000,800); t=time.time(); ts.extremal_tilings(d); print('domino extremal rect 1000x800', time.time()-t)
" > gpurun_out/r2_extremal_time.txt 2>&1
python -m pytest tests/test_lozenge_gpu.py tests/test_domino_gpu.py tests/test_heights_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t4.log
for t in racecheck; do timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py cftp heights strips domain loz > gpurun_out/san2_${t}.log 2>&1; done
python tools/probe_host_copies.py > gpurun_out/r2_hostcopies.json 2>&1
python tools/make_warm_state.py bench_data/aztec4096_warm.npz > gpurun_out/r2_warm_trace.jsonl 2>&1
cp bench_data/aztec4096_warm.npz gpurun_out/

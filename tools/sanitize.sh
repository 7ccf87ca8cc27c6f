#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over every kernel family
# and TSB_* kernel variant on small lattices (tools/sanitize_run.py checks each
# result against the oracle).  Summary: gpurun_out/sanitizer.txt
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitizer.txt
mkdir -p gpurun_out
: > $OUT
run() {  # tool env... -- workload
    local tool=$1; shift
    local envs=()
    while [ "$1" != "--" ]; do envs+=("$1"); shift; done
    shift
    local log=gpurun_out/san_${tool}_$(echo "$*_${envs[*]}" | tr ' =' '__').log
    env "${envs[@]}" timeout 900 compute-sanitizer --tool $tool --error-exitcode 3 python tools/sanitize_run.py "$@" \
        > "$log" 2>&1
    local rc=$?
    echo "$tool [$*] ${envs[*]:-default}: rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' "$log" | tail -1) $(grep -h ' ok$' "$log" | tr '\n' ' ')" | tee -a $OUT
}
for tool in memcheck synccheck racecheck; do
    run $tool -- domino
    run $tool TSB_DOM_WPL=1 -- domino
    run $tool TSB_DOM_PIPE=1 -- domino
    run $tool TSB_DOM_RESIDENT=1 -- domino
    run $tool TSB_DOM_RESIDENT=0 TSB_DOM_ADAPT=0 -- domino
    run $tool TSB_DOM_COLLAPSE=0 -- domino
    run $tool -- cftp heights strips domain
    run $tool TSB_DOM_RESIDENT=0 -- cftp
    run $tool -- sv
    run $tool TSB_SV_K=2 TSB_SV_NW=8 -- sv
    run $tool TSB_SV_WPL=1 -- sv
    run $tool TSB_SV_DENSE=1 -- sv
    run $tool TSB_SV_COLLAPSE=0 -- sv
    run $tool -- loz
    run $tool TSB_LZ_K=2 -- loz
    run $tool TSB_LZ_DENSE=1 -- loz
    run $tool TSB_LZ_COLLAPSE=0 -- loz
done

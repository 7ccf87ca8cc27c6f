#!/usr/bin/env python
"""Copy a tools/gpu_round2_final.sh run (gpurun_out/final/) into the committed
profiles/round2_*: bench lines, config throughputs, C5 full samples, height
export timings, GPU test tail, smoke, sanitizer log, ncu summaries and the
launch list of the bench step."""
import collections
import csv
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F, P = os.path.join(ROOT, "gpurun_out", "final"), os.path.join(ROOT, "profiles")

COPIES = {
    "bench.json": "round2_bench.json",
    "bench_ref.json": "round2_bench_reference.json",
    "bench_2ranks.json": "round2_bench_2ranks_shared_gpu.json",
    "configs_plain.jsonl": "round2_configs_plain.jsonl",
    "configs_collapsed.jsonl": "round2_configs_collapsed.jsonl",
    "c5full8.jsonl": "round2_c5_full8.jsonl",
    "c5full64.jsonl": "round2_c5_full64.jsonl",
    "heights.jsonl": "round2_heights.jsonl",
    "pytest_gpu.txt": "round2_pytest_gpu.txt",
    "smoke.txt": "round2_smoke.txt",
    "sanitizer.txt": "round2_sanitizer.txt",
}
NCU = ["prof_multi", "prof_multi_warm", "prof_multi_warm_collapsed", "prof_sv", "prof_lz", "prof_pipe"]
JSONL = {"configs_plain.jsonl", "configs_collapsed.jsonl", "c5full8.jsonl", "c5full64.jsonl", "heights.jsonl"}


def json_lines(path):
    return [ln for ln in open(path).read().splitlines() if ln.startswith("{")]


def main():
    for src, dst in COPIES.items():
        s = os.path.join(F, src)
        if not os.path.exists(s):
            print("missing", src)
            continue
        if src.endswith(".json") or src in JSONL:
            lines = json_lines(s)
            if src.endswith(".json"):
                lines = lines[-1:]
            open(os.path.join(P, dst), "w").write("\n".join(lines) + "\n")
        else:
            shutil.copy(s, os.path.join(P, dst))
    for r in NCU:
        s = os.path.join(F, f"{r}_ncu.txt")
        if os.path.exists(s):
            shutil.copy(s, os.path.join(P, f"round2_{r}_ncu.txt"))
    rows = [r for r in csv.reader(open(os.path.join(F, "launches_4096.csv"))) if len(r) > 10]
    h = rows[0]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        agg[r[iK]][r[iM]].append(float(r[iV].replace(",", "")))
    unit = {}
    iU = h.index("Metric Unit")
    for r in rows[1:]:
        unit[r[iM]] = r[iU]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
    tscale = scale.get(unit.get("gpu__time_duration.sum", "ns"), 1e-3)
    bscale = {"byte": 1e-3, "Kbyte": 1.0, "Mbyte": 1e3, "Gbyte": 1e6}
    tot = sum(sum(v["gpu__time_duration.sum"]) for v in agg.values()) * tscale
    out = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 150",
           "#   python bench.py --order 4096 --steps 2 --warmup 1 --sweeps-per-step 128 --no-e2e --no-cpu-baseline --no-warm --no-collapsed",
           "# per-launch times are serialised and cold (ncu flushes caches per kernel); the multi-sweep kernel's SHARE of the step is the evidence",
           "# (the FillFunctor kernel is bench.py's 256 MiB L2 flush between timed steps, outside the CUDA events)"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
        tt = [x * tscale for x in v["gpu__time_duration.sum"]]
        rd = [x * bscale.get(unit.get("dram__bytes_read.sum", "Kbyte"), 1.0) for x in v.get("dram__bytes_read.sum", [0])]
        wr = [x * bscale.get(unit.get("dram__bytes_write.sum", "Kbyte"), 1.0) for x in v.get("dram__bytes_write.sum", [0])]
        name = k.split("(")[0][:70]
        out.append(f"{name:70s} launches={len(tt):5d} total_us={sum(tt):9.1f} share={sum(tt) / tot:6.3f} "
                   f"avg_us={sum(tt) / len(tt):8.2f} dram_KB_per_launch={(sum(rd) + sum(wr)) / len(tt):10.1f}")
    open(os.path.join(P, "round2_launches_4096.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()

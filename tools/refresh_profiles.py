#!/usr/bin/env python
"""Copy a tools/gpu_round.sh run (gpurun_out/) into the committed profiles/:
bench lines, config throughputs, ncu summaries, launch list, traffic.json."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
A = "--order 4096 --steps 2 --warmup 1 --sweeps-per-step 128 --no-e2e --no-cpu-baseline"


def last_json(f):
    return [ln for ln in open(os.path.join(G, f)).read().splitlines() if ln.startswith("{")][-1]


def summ(rep, cmd, out, note):
    s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), os.path.join(G, rep), "--sass",
                        "25"], capture_output=True, text=True).stdout
    open(os.path.join(P, out), "w").write(f"# {note}\n# command: {cmd}\n" + s)
    return s


def main():
    open(os.path.join(P, "round1_bench.json"), "w").write(last_json("bench.txt") + "\n")
    open(os.path.join(P, "round1_bench_reference.json"), "w").write(last_json("bench_ref.txt") + "\n")
    cfg = [ln for ln in open(os.path.join(G, "configs.txt")).read().splitlines() if ln.startswith("{")]
    open(os.path.join(P, "round1_configs.jsonl"), "w").write("\n".join(cfg) + "\n")
    s = summ("prof_multi_warm.ncu-rep",
             f"ncu --set full --clock-control none --cache-control none --import-source on -k regex:domino_multi -s 100 -c 2 python bench.py {A}",
             "round1_domino_multi_ncu.txt",
             "domino_multi_kernel<0> (2 sweeps/launch, band-aligned tiles), Aztec 4096 from T_max, warm L2 "
             "(state resident between launches, as in the graph replays)")
    summ("prof_sv_warm.ncu-rep",
         "ncu --set full --clock-control none --cache-control none --import-source on -k regex:sv_multi -s 200 -c 1 python tools/prof_driver.py sv",
         "round1_sv_multi_ncu.txt", "sv_multi_kernel<3,16> (8 class sweeps/launch), six-vertex DWBC n=2048 Delta=1/2 after 2000 sweeps from h_min")
    summ("prof_lz_warm.ncu-rep",
         "ncu --set full --clock-control none --cache-control none --import-source on -k regex:lz_multi -s 200 -c 1 python tools/prof_driver.py lz",
         "round1_lz_multi_ncu.txt", "lz_multi_kernel<0> (4 sweeps/launch, band-aligned tiles), lozenge hexagon 1000^3 q=0.999 after 2000 sweeps from T_min")
    if os.path.exists(os.path.join(G, "prof_multi_pipe.ncu-rep")):
        summ("prof_multi_pipe.ncu-rep",
             "ncu --set full --clock-control none --cache-control none --import-source on -k regex:domino_multi_pipe -s 20 -c 1 python tools/dbg_sizes.py 16384",
             "round1_domino_multi_pipe_ncu.txt",
             "domino_multi_pipe_kernel<0> (2 sweeps/launch, persistent blocks, next tile fetched by cp.async), C4 lattice "
             "Aztec 16384 from T_max after 256 sweeps (HBM-streaming: 2 x 285 MB state buffers)")
    if os.path.exists(os.path.join(G, "configs_extra.txt")):
        extra = [ln for ln in open(os.path.join(G, "configs_extra.txt")).read().splitlines() if ln.startswith("{")]
        strips = [ln for ln in extra if json.loads(ln)["config"].startswith("strips")]
        batched = [ln for ln in extra if not json.loads(ln)["config"].startswith("strips")]
        if strips:
            open(os.path.join(P, "round1_strips_compute.jsonl"), "w").write("\n".join(strips) + "\n")
        if batched:
            open(os.path.join(P, "round1_batched.jsonl"), "w").write("\n".join(batched) + "\n")
    # traffic of the hot kernel: launch 1 of the --set full capture
    vals = {}
    for ln in s.splitlines():
        parts = ln.split()
        if parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum"):
            unit, v = parts[1], float(parts[2])
            vals[parts[0]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "sector": 32}.get(unit, 1)
    t = json.load(open(os.path.join(P, "traffic.json")))
    t["domino_multi_kernel"] = {
        "dram_bytes_per_launch": int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]),
        "lts_bytes_per_launch": int(vals["lts__t_sectors.sum"]), "sweeps_per_launch": 2,
        "source": "profiles/round1_domino_multi_ncu.txt: ncu --set full --cache-control none, launch 1 of 2 "
                  "(dram__bytes_read.sum + dram__bytes_write.sum; lts__t_sectors.sum x 32 B)",
        "note": "Aztec 4096: the state planes stay L2-resident across the graph replays (algorithmic: 67.2 MB per launch)"}
    json.dump(t, open(os.path.join(P, "traffic.json"), "w"), indent=1)
    rows = [r for r in csv.reader(open(os.path.join(G, "launches_4096.csv"))) if len(r) > 10]
    h = rows[0]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        agg[r[iK]][r[iM]].append(float(r[iV].replace(",", "")))
    tot = sum(sum(v["gpu__time_duration.sum"]) for v in agg.values())
    lines = ["# ncu launch list (gpu__time_duration, dram bytes; --cache-control none --clock-control none), "
             "Aztec 4096 bench step of 128 sweeps",
             "# command: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum "
             f"--clock-control none --cache-control none -s 200 -c 200 --csv python bench.py {A}",
             "kernel, launches, mean_ns, share_of_time, mean_dram_read_B, mean_dram_write_B"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
        tt, rd, wr = v["gpu__time_duration.sum"], v.get("dram__bytes_read.sum", [0]), v.get("dram__bytes_write.sum", [0])
        lines.append(f"{k.split('(')[0]}, {len(tt)}, {sum(tt) / len(tt):.0f}, {sum(tt) / tot:.3f}, "
                     f"{sum(rd) / len(rd):.0f}, {sum(wr) / len(wr):.0f}")
    open(os.path.join(P, "round1_launches_4096.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    print(json.dumps(t["domino_multi_kernel"]))


if __name__ == "__main__":
    main()

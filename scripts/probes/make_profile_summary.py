"""Regenerate profiles/ncu_summary.json and profiles/rNN_launches.md from a
gpu_round.sh run (gpurun_out/launches.csv, gpurun_out/prof_bench.ncu-rep,
gpurun_out/bench.json).  Usage: python scripts/make_profile_summary.py 01"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rnd = sys.argv[1] if len(sys.argv) > 1 else "01"
out = os.path.join(ROOT, "gpurun_out")

rows = list(csv.reader(open(os.path.join(out, "launches.csv"))))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg, n = collections.OrderedDict(), collections.Counter()
for r in data:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].strip()
    sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
    agg[name] = agg.get(name, 0.0) + float(r[vi].replace(",", "")) * sc
    n[name] += 1
tot = sum(agg.values())
lines = ["| share | total us | launches | kernel |", "|---:|---:|---:|---|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    lines.append(f"| {100 * v / tot:.2f}% | {v:.1f} | {n[k]} | `{k}` |")
open(os.path.join(ROOT, "profiles", f"r{rnd}_launches.md"), "w").write(
    "Launch list of `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu` (plan setup + 3 outer\n"
    "iterations, the first one cold) from `ncu --metrics gpu__time_duration.sum --clock-control none`\n"
    "(cold-cache, serialised: compare shares).\n\n" + "\n".join(lines) + "\n")

raw = subprocess.run(["ncu", "-i", os.path.join(out, "prof_bench.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, v = rr[0], rr[2]
g = lambda m: float(v[h.index(m)].replace(",", ""))
bench = json.load(open(os.path.join(out, "bench.json")))
summ = {
    "round": int(rnd), "kernel": v[h.index("Kernel Name")].split("(")[0],
    "capture": "ncu --set full --clock-control none --import-source on -k regex:svt_subspace -s 2 -c 1 on "
               "`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu` (a warm ADMM iteration, config 2)",
    "duration_ms": g("gpu__time_duration.sum"),
    "dram_read_bytes": g("dram__bytes_read.sum") * 1e6, "dram_write_bytes": g("dram__bytes_write.sum") * 1e6,
    "svt_dram_bytes_per_launch": (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) * 1e6,
    "algorithmic_bytes_per_launch": 512 * (16 * 242 * 120 + 16 * 8 * 256),
    "sm_throughput_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "fma_pipe_active_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": g("launch__registers_per_thread"),
    "smem_per_block_kb": g("launch__shared_mem_per_block_dynamic"),
    "shared_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "bench": {k: bench[k] for k in ("value", "ms_per_step")} | {"svt_ms": bench["hankel_svt"]["kernel_ms"],
                                                              "roofline_frac": bench["roofline"]["frac"],
                                                              "e2e": bench["e2e"]["value"]},
}
json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps(summ, indent=1))
print("\n".join(lines[:10]))

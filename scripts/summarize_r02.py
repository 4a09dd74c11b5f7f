"""Summaries of the round-2 captures (scripts/gpu_profiles_r02.sh) into
profiles/r02_*: the launch list of the headline bench and, per captured
kernel, the counters the roofline and the verdict ask for."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__waves_per_multiprocessor",
    "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]
CAPS = {
    "c2_svt": "config 2 (headline): svt_subspace_kernel<120,48,32> warm iteration, 512 lifted 242x120",
    "c2_cols": "config 2: k_spirit_cols (SPIRiT column stage inside the CG loop)",
    "sv_tall": "SHLR-SV headline geometry: svt_subspace_kernel<248,48,32,BIG> (512 tall weighted 242x240)",
    "huge": "config 5 point 498x480: svt_subspace_kernel<496,32,16,HUGE> (1024 matrices, cold)",
    "smalld": "config 5 point 250x56: svt_subspace_kernel<56,16,32> (512 matrices, cold)",
}


def raw(name):
    rows = list(csv.reader(open(os.path.join(OUT, f"prof_{name}.raw.csv"))))
    h, units, v = rows[0], rows[1], rows[2]
    out = {"kernel": v[h.index("Kernel Name")]}
    for m in METRICS:
        if m in h:
            val = v[h.index(m)].replace(",", "")
            try:
                out[m] = float(val)
            except ValueError:
                out[m] = val
            out[m + ".unit"] = units[h.index(m)]
    return out


def main():
    summ = {}
    for name, what in CAPS.items():
        p = os.path.join(OUT, f"prof_{name}.raw.csv")
        if os.path.exists(p) and os.path.getsize(p) > 1000:
            summ[name] = dict(raw(name), what=what)
    json.dump(summ, open(os.path.join(PROF, "r02_ncu_summary.json"), "w"), indent=1)
    for name in summ:
        hot = os.path.join(OUT, f"prof_{name}.hot.txt")
        if os.path.exists(hot) and os.path.getsize(hot) > 0:
            subprocess.run(["cp", hot, os.path.join(PROF, f"r02_prof_{name}.hot.txt")])
    tab = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_table.py"),
                          os.path.join(OUT, "launches.csv")], capture_output=True, text=True).stdout
    subprocess.run(["cp", os.path.join(OUT, "launches.csv"), os.path.join(PROF, "r02_ncu_launches.csv")])
    open(os.path.join(PROF, "r02_launches.md"), "w").write(
        "Launch list of `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra` (plan setup\n"
        "+ 3 outer iterations of config 2, the first one cold) from `ncu --metrics gpu__time_duration.sum\n"
        "--clock-control none` (cold-cache, serialised launches: compare shares, not absolute times).\n"
        "`k_fma_probe` is the bench's FP32 peak measurement, not part of the step: without it the SVT kernel's\n"
        "share of the listed time is its share of the step (bench: `hankel_svt.share_of_step`).\n\n" + tab)
    for k, v in summ.items():
        print(k, {m.split(".")[0][:40]: v.get(m) for m in METRICS[:9]})


if __name__ == "__main__":
    main()

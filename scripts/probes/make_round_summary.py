"""Write profiles/rNN_summary.md from profiles/rNN_bench.json, the cold and warm
launch lists and profiles/ncu_summary.json.  Usage: make_round_summary.py 01"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rnd = sys.argv[1] if len(sys.argv) > 1 else "01"
P = os.path.join(ROOT, "profiles")
b = json.load(open(os.path.join(P, f"r{rnd}_bench.json")))
n = json.load(open(os.path.join(P, "ncu_summary.json")))


def table(csv):
    return subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_table.py"), csv],
                          capture_output=True, text=True).stdout


o = b.get("other_workloads", {})
e2e = b["e2e"]
txt = f"""# Round {int(rnd)} profile summary (B200, sm_100a)

Bench line (`python bench.py`, default 20 steps / 3 warm-up, config 2, `profiles/r{rnd}_bench.json`):
`value` {b['value']:.1f} iterations/s ({b['ms_per_step']:.2f} ms/iter); e2e {e2e['value']:.1f} iterations/s
(median of three 50-iteration public-API calls with host buffers), {e2e.get('with_device_calibration', {}).get('value', float('nan')):.1f}
with the SPIRiT calibration on the device inside the timed call; Hankel-SVT {b['hankel_svt']['kernel_ms']:.2f} ms
({b['hankel_svt']['matrices_per_s'] / 1e3:.1f} k matrices/s); roofline {b['roofline']['achieved']:.1f} TFLOP/s algorithmic =
{100 * b['roofline']['frac']:.1f} % of the measured FP32 peak ({b['roofline']['peak']:.1f} TFLOP/s); SM clock
{b['clocks']['sm_mhz']:.0f} MHz, throttle reasons {b['clocks']['reasons']}; reference CPU (oracle/_ref, 1 core)
{b['cpu_baseline']['value']:.4f} iterations/s.  (Round start: 208 it/s, SVT 3.94 ms, 23.6 % of peak.)

Side workloads in the same line: config 4 {o.get('config4_param', {}).get('value', float('nan')):.1f} it/s over 256 FE slices
(e2e {o.get('config4_param', {}).get('e2e', {}).get('value', float('nan')):.1f}); config 3 {o.get('config3_large_d', {}).get('value', float('nan')):.1f} it/s over
its 50 iterations; config-5 sweep points in `other_workloads.config5_sweep`.

## Launch list (`r{rnd}_ncu_launches.csv`)

`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` on
`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu` (plan setup + 3 outer iterations, the first one
cold; default cache control, i.e. caches flushed per kernel: compare shares, not absolute times):

{table(os.path.join(P, f'r{rnd}_ncu_launches.csv'))}
Same command with `--cache-control none` (warm L2, as in the graph-launched loop;
`r{rnd}_ncu_launches_warm.csv`):

{table(os.path.join(P, f'r{rnd}_ncu_launches_warm.csv'))}
## Full capture of the SVT kernel (`ncu_summary.json`)

`ncu --set full --clock-control none --import-source on -k regex:svt_subspace -s 2 -c 1` on the same
command (a warm iteration): {n['duration_ms']:.2f} ms; DRAM {n['dram_read_bytes'] / 1e6:.0f} MB read +
{n['dram_write_bytes'] / 1e6:.0f} MB written = {n['svt_dram_bytes_per_launch'] / 1e6:.0f} MB per launch (algorithmic
{n['algorithmic_bytes_per_launch'] / 1e6:.0f} MB: the duals are read and written once, nothing re-read); FMA pipe
{n['fma_pipe_active_pct']:.1f} % active; issue slots {n['issue_active_pct']:.1f} % active; {n['registers_per_thread']:.0f}
registers, {n['smem_per_block_kb']:.0f} KB smem, 1 CTA (16 warps) per SM.  Phase clocks: DESIGN.md §4.

## Side workloads
* `r{rnd}_param_launches.md`, `ncu_side_summary.json` (`prof_param_pe`, `prof_param_echo`): config 4.
* `r{rnd}_c3_launches.md`, `ncu_side_summary.json` (`prof_c3`): config 3 (large-d levels).
* `r{rnd}_param_pe_hot.txt`, `r{rnd}_c3_hot.txt`: top source lines by warp-stall samples.
"""
open(os.path.join(P, f"r{rnd}_summary.md"), "w").write(txt)
print(txt[:1500])

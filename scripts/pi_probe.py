"""Config-2 plan probe: per-iteration sweeps (warm start) and SVT timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_11650_b200 import api as A
y, mask, g, hcfg = bench.make_inputs()
warm = int(os.environ.get("WARM", 1))
acfg = A.AdmmConfig(max_outer=50, tol=1e-300, enable_spirit=True)
plan = A.PiPlan(y, mask, g, hcfg, acfg)
plan.set_warm_start(bool(warm))
plan.set_timing(True)
iters = int(os.environ.get("ITERS", 12))
for it in range(iters):
    plan.run(1); plan.sync()
    svt_ms, tot, _ = plan.timing()
    sw = plan.debug_sweeps()
    s1, s2 = sw // 100, sw % 100
    hist = np.bincount(sw % 100, minlength=21)[:21]
    print("   sweep histogram:", " ".join(f"{i}:{c}" for i, c in enumerate(hist) if c))
    print(f"iter {it+1}: svt {svt_ms:.2f} ms total {tot:.2f} ms | stage1 mean {s1.mean():.2f} max {s1.max()} | stage2 mean {s2.mean():.2f} max {s2.max()}", flush=True)
if os.environ.get("SHLR_PHASE_CLK"):
    ph = plan.debug_phases().astype(np.float64)
    ok = ph[:, 7] > 0
    d = lambda a, b: (ph[ok, b] - ph[ok, a]) / 1e3
    print(f"phase kcycles (mean over {ok.sum()} matrices): start {d(0,3).mean():.0f} [pass {ph[ok,1].mean()/1e3:.0f} qr {ph[ok,2].mean()/1e3:.0f}] "
          f"H-pass {d(3,4).mean():.0f} RR-jacobi {d(4,5).mean():.0f} VU {d(5,6).mean():.0f} Z-pass {d(6,7).mean():.0f} total {d(0,7).mean():.0f}")
    print("pass split kcycles: wait %.0f build %.0f gemm1 %.0f sum %.0f gemm2 %.0f" % tuple(ph[ok, 8 + i].mean() / 1e3 for i in range(5)))
    e = [(ph[ok, 17 + i] - ph[ok, 16 + i]).mean() / 1e3 for i in range(6)]
    print("RR split kcycles: tridiag %.0f similarity %.0f bisection %.0f twisted+clusters %.0f mgs %.0f backtransform %.0f" % tuple(e))
    print("QR split kcycles (Cholesky QR): gram+scale %.0f cholesky %.0f inverse %.0f product %.0f" % tuple(ph[ok, i].mean() / 1e3 for i in (13, 14, 15, 23)))
    tot = d(0, 7)
    print("total kcycles percentiles 50/90/99/max:", np.percentile(tot, [50, 90, 99]).round(0), tot.max().round(0),
          "| RR max", d(4, 5).max().round(0), "| matrices stamped", int(ok.sum()))

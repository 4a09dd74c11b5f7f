# Accuracy / speed of subspace-solver variants on config 2 (image vs the
# reference's 50-iteration run; SVT time and phase cycles of a warm launch).
run() {
  echo "== $*"
  env "$@" SV=0 timeout 200 python scripts/c2_check.py
  env "$@" SHLR_PHASE_CLK=1 ITERS=3 timeout 120 python scripts/probes/pi_probe.py | grep -v histogram | tail -n 3
}
run SHLR_Q_WARM=2
run SHLR_Q_WARM=2 SHLR_INNER_NORM=1
run SHLR_Q_WARM=3 SHLR_INNER_NORM=1
run SHLR_Q_WARM=1

# RR-tolerance sweep on config 2: parity of the 50-iteration image vs the
# reference run and the Rayleigh-Ritz sweep histogram / phase cycles.
for cfg in "2e-6 1e-7 0" "2e-6 1e-6 0" "1e-5 1e-6 0" "1e-5 1e-5 0" "2e-6 1e-7 0.5"; do
  set -- $cfg
  echo "== RR rel=$1 abs=$2 tail=$3"
  SHLR_RR_REL=$1 SHLR_RR_ABS=$2 SHLR_RR_TAIL=$3 SV=0 timeout 200 python scripts/c2_check.py
  SHLR_RR_REL=$1 SHLR_RR_ABS=$2 SHLR_RR_TAIL=$3 SHLR_PHASE_CLK=1 ITERS=4 timeout 120 python scripts/probes/pi_probe.py | tail -n 3
done

# warps x barrier-cost sweep of the lane-SIMT kernel on C3 (one JSON summary line each)
for rep in 1 2; do for w in 6 8 10 12; do for b in 150 200 300; do
  BENCH_ARGS="--warps $w" bash tools/knob_sweep.sh "EMTB200_CG_BARRIER=$b W=$w"
done; done; done

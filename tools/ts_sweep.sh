# task-SIMT vs lane-SIMT timing on every workload
for wl in c2 c3 c5 c4; do
  BENCH_ARGS="--workload $wl" bash tools/knob_sweep.sh "K=specialised"
  for w in 2 4 8; do BENCH_ARGS="--workload $wl --warps $w" bash tools/knob_sweep.sh "EMTB200_KERNEL=tsimt W=$w"; done
done

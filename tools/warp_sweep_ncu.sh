# Warp-count sweep + ncu source-level capture of the C2 and C3 specialised kernels.
set -x
for w in 4 6 8 10 12 16; do BENCH_ARGS="--warps $w" bash tools/knob_sweep.sh "X=$w"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:emt_cg_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu_c2b python bench.py --workload c2 --skip-cpu --skip-e2e --steps 1 --emt-steps 200 > gpurun_out/ncu_c2b.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:emt_cg_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu_c3b python bench.py --skip-cpu --skip-e2e --steps 1 --emt-steps 200 > gpurun_out/ncu_c3b.log 2>&1
ls -la gpurun_out/

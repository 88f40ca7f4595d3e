#!/bin/bash
# Round profile on the GPU box:  tools/prof_round.sh <tag>
# Default bench line (C3, with e2e + e2e_cold + cpu_baseline + parity), the reference arm, C2/C4/C5/scale,
# the launch list of the default command and one full ncu capture of the step-loop kernel.
t=${1:-r2a}
timeout 900 python bench.py > gpurun_out/bench_${t}.json 2> gpurun_out/bench_${t}.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_${t}_reference.json 2> gpurun_out/bench_${t}_reference.err
for w in c2 c4 c5 scale; do timeout 900 python bench.py --workload $w > gpurun_out/bench_${t}_$w.json 2> gpurun_out/bench_${t}_$w.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${t}.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:emt_cg_kernel --launch-skip 3 -c 1 \
    -o gpurun_out/ncu_${t} python bench.py --skip-cpu --skip-e2e --steps 1 --emt-steps 200 > gpurun_out/ncu_${t}.log 2>&1
for f in gpurun_out/bench_${t}*.json; do echo "$f"; head -c 300 "$f"; echo; done

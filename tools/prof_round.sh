# Round profile: default bench line (C3), C2/C4/C5 (+ tensor-core C5), launch list, one full ncu capture.
timeout 600 python bench.py > gpurun_out/bench_r1o.json 2> gpurun_out/bench_r1o.err
for w in c2 c4 c5; do timeout 600 python bench.py --workload $w > gpurun_out/bench_r1o_$w.json 2> gpurun_out/bench_r1o_$w.err; done
timeout 600 python bench.py --workload c5 --tensor-solve > gpurun_out/bench_r1o_c5t.json 2> gpurun_out/bench_r1o_c5t.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1o.csv python bench.py --steps 2 --warmup 3 --skip-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:emt_cg_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu_r1o python bench.py --skip-cpu --skip-e2e --steps 1 --emt-steps 200 > gpurun_out/ncu_r1o.log 2>&1
cat gpurun_out/bench_r1o.json

# Round profile: default bench line, other workloads, launch list, one full ncu capture.
timeout 600 python bench.py > gpurun_out/bench_r1h.json 2> gpurun_out/bench_r1h.err
for w in c2 c4 c5; do timeout 600 python bench.py --workload $w > gpurun_out/bench_r1h_$w.json 2> gpurun_out/bench_r1h_$w.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1h.csv python bench.py --steps 2 --warmup 3 --skip-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:emt_cg_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu_r1h python bench.py --skip-cpu --skip-e2e --steps 1 --emt-steps 200 > gpurun_out/ncu_r1h.log 2>&1
cat gpurun_out/bench_r1h.json

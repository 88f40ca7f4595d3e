set -x
for k in generic; do timeout 300 python bench.py --workload c2 --kernel $k --skip-cpu --skip-e2e --steps 5 > gpurun_out/c2_$k.json 2>&1; done
for w in 1 2 4 8; do timeout 300 python bench.py --workload c2 --warps $w --skip-cpu --skip-e2e --steps 5 > gpurun_out/c2_w$w.json 2>&1; done
for w in 4 8 12 16; do timeout 300 python bench.py --workload c3 --warps $w --skip-cpu --skip-e2e --steps 5 > gpurun_out/c3_w$w.json 2>&1; done
timeout 300 python bench.py --workload c3 --kernel generic --skip-cpu --skip-e2e --steps 5 > gpurun_out/c3_generic.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:emt_cg_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu_c2 python bench.py --workload c2 --skip-cpu --skip-e2e --steps 1 --emt-steps 200 > gpurun_out/ncu_c2.log 2>&1
for f in gpurun_out/c2_*.json gpurun_out/c3_*.json; do echo $f; grep -o '"value": [0-9.e+]*' $f | head -1; grep -o '"kernel": "[^"]*"' $f; done

# Multi-rank control flow of bench.py on ONE GPU (2 ranks share it, gloo collectives).
export BENCH_DIST_BACKEND=gloo BENCH_SHARE_GPU=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --emt-steps 100 --skip-cpu 2>&1 | grep -v "^W\|Warning\|warn" | tail -3 | cut -c1-400
timeout 600 $R bench.py --gpus 2 --workload c4 --steps 2 --warmup 3 --emt-steps 100 --skip-cpu 2>&1 | grep -v "^W\|Warning\|warn" | tail -3 | cut -c1-400
timeout 600 $R bench.py --gpus 2 --impl reference --steps 2 --warmup 3 --cpu-emt-steps-per-step 20 2>&1 | tail -2 | cut -c1-300
timeout 600 $R bench.py --gpus 2 --workload scale --scenarios 32 --steps 2 --warmup 3 --emt-steps 20 --skip-cpu 2>&1 | grep -v "^W\|Warning\|warn" | tail -3 | cut -c1-400

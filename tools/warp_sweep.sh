for rep in 1 2; do for w in c3 c2; do for k in 4 6 8; do
out=$(timeout 300 python bench.py --workload $w --skip-e2e --skip-cpu --steps 10 --warps $k 2>/dev/null)
python -c "import json,sys; d=json.loads(sys.argv[1]); print('$w warps=$k', round(d['ms_per_step'],4), d['kernel'][:120])" "$out"
done; done; done

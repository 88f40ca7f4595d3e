# warps per lane group A/B: bash tools/warp_sweep.sh "c3 c2" "4 6 8"
wls=${1:-"c3 c2"}; ks=${2:-"4 6 8"}
for rep in 1 2; do for w in $wls; do for k in $ks; do
out=$(timeout 300 python bench.py --workload $w --skip-e2e --skip-cpu --steps 10 --warps $k 2>/dev/null)
python -c "import json,sys; d=json.loads(sys.argv[1]); print('$w warps=$k', round(d['ms_per_step'],4), d['kernel'][:120])" "$out"
done; done; done

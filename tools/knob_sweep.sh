# Times the C3 bench under code-generator knob settings (one JSON line each).
# usage: bash tools/knob_sweep.sh "ENV=.. ENV=.." "ENV=.." ...
for cfg in "$@"; do
  out=$(env $cfg timeout 300 python bench.py --skip-cpu --skip-e2e --steps 10 ${BENCH_ARGS} 2>/dev/null | tail -1)
  echo "$cfg :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["kernel"][:90])' 2>/dev/null)"
done

#!/bin/bash
# A/B timing of generator knobs on the GPU box with a developer build:
#   tools/ab.sh "c3 c2" "" "EMTB200_CG_DIVGUARD=0" ...
# Each argument after the workload list is one environment setting ("" = defaults);
# every (setting, workload) pair runs bench.py once (no e2e, no cpu leg).
python paper_1903_01081_b200/build.py --dev > /dev/null 2>&1
wls=$1; shift
for rep in 1 2; do
for cfg in "$@"; do
  for w in $wls; do
    out=$(env $cfg python bench.py --workload $w --skip-e2e --skip-cpu --allow-dev-build --steps 10 2>/dev/null)
    python -c "
import json,sys; d=json.loads(sys.argv[1]); print('$w', '[$cfg]', round(d['ms_per_step'],4), d['unit'], d['value'])" "$out"
  done
done
done

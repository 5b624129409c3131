#!/bin/bash
# A/B of environment overrides on one box, twice each: bench ms/step, gather
# ms, ring depth, row tile.   CFG=4 bash tools/ab_env.sh "X=0" "LMKAN_B200_DUP16=0" ...
for rep in 1 2; do
for e in "$@"; do
  echo -n "cfg${CFG:-2} $e: "
  env $e timeout 300 python bench.py --config ${CFG:-2} --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['kernel_plan']; print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), 'nbuf', p['nbuf'], 'rows', p['rows_per_cta'], 'ot', p['out_tile'], p['mode'])"
done; done

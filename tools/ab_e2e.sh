#!/bin/bash
# e2e (host-buffer) samples/s under environment overrides, twice each:
#   CFG=2 bash tools/ab_e2e.sh "X=0" "LMKAN_B200_HOST_CHUNKS=12" ...
for rep in 1 2; do
for e in "$@"; do
  echo -n "cfg${CFG:-2} $e: "
  env $e timeout 300 python bench.py --config ${CFG:-2} --no-cpu-baseline $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(e['value']/1e6,3), 'M/s', round(e['ms_per_step'],3), 'ms', e.get('steps'), 'steps; dropin', round((d.get('e2e_dropin') or {}).get('value',0)/1e6,3))"
done; done

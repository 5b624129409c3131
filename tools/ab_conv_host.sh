#!/bin/bash
# cfg4 host-entry (e2e) A/B over the conv chunking knobs:
#   bash tools/ab_conv_host.sh "LMKAN_B200_CONV_CHUNK_ROWS=512" "LMKAN_B200_HOST_TAPER=1" ...
for rep in 1 2; do
for e in "$@"; do
  echo -n "cfg4 $e: "
  env $e timeout 300 python bench.py --config 4 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],4), 'e2e', '%.4g' % d['e2e']['value'])"
done; done

#!/bin/bash
# A/B of env toggles on bench lines (ms/step, gather-kernel ms, smem frac, e2e M samples/s):
#   VAR=LMKAN_B200_PIXREC VALS="0 1" CFGS="4" bash tools/ab_pixrec.sh
for rep in 1 2; do for c in ${CFGS:-4}; do for v in ${VALS:-0 1}; do echo -n "cfg$c $VAR=$v "; env $VAR=$v timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['smem_gather_ceiling']['frac'],3), round(d['e2e']['value']/1e6,2))"; done; done; done

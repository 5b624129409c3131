#!/bin/bash
# A/B timing on one box: bench ms/step (and gather-kernel ms) of a baseline
# build (ablib/liblmkan_b200_base.so, built from an earlier commit) against the
# in-tree build, alternating twice. CFGS="2 5" EXTRA_ENV="LMKAN_B200_PAIR_BLOCK=256"
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then export LMKAN_B200_LIB=$PWD/ablib/liblmkan_b200_base.so; else unset LMKAN_B200_LIB; fi
  for c in ${CFGS:-2 5}; do A=""; [ $c = 5 ] && A="--shards 8 --steps 5"
    env $EXTRA_ENV timeout 300 python bench.py --config $c $A --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg$c', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"
  done; done; done

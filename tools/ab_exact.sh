#!/bin/bash
# Same-box A/B of the reference-precision (fp64, bit-identical) forward: a
# baseline build (ablib/liblmkan_b200_base.so) against the in-tree build.
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then export LMKAN_B200_LIB=$PWD/ablib/liblmkan_b200_base.so; else unset LMKAN_B200_LIB; fi
  timeout 300 python bench.py --precision 64 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v exact cfg2', round(d['ms_per_step'],3), '%.4g' % d['value'])"
done; done

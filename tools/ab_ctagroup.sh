#!/bin/bash
# CTA-order group sweep (choose_cta_group / LMKAN_B200_CTA_GROUP): bench ms and
# the gather kernel's DRAM reads (ncu, one launch) per group.
#   CTA_GROUPS="1 2 4" CFGS="2 5" bash tools/ab_ctagroup.sh
mkdir -p gpurun_out
O=gpurun_out/ctagroup.txt
for cfg in ${CFGS:-2 5}; do
  a=""; [ $cfg = 5 ] && a="--shards 8"
  envs=""; for g in ${CTA_GROUPS:-1 2 4}; do envs="$envs LMKAN_B200_CTA_GROUP=$g"; done
  CFG=$cfg BENCH_ARGS="$a" bash tools/ab_env.sh $envs >> $O 2>&1
  for g in ${CTA_GROUPS:-1 2 4}; do
    LMKAN_B200_CTA_GROUP=$g timeout 600 ncu --metrics dram__bytes_read.sum --clock-control none \
      -k regex:fwd_fused -s 3 -c 1 --csv python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $a 2>/dev/null \
      | grep -E "dram__" | awk -F'","' -v c=$cfg -v g=$g '{gsub(/"/,"",$NF); print "cfg" c " group " g " dram_read_bytes " $NF}' >> $O
  done
done

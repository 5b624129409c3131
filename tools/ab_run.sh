#!/bin/bash
# A/B timing of library builds on one box: tools/ab/<name>/liblmkan_b200.so
# VARS="a b" CFGS="2 3" bash tools/ab_run.sh
for c in ${CFGS:-2}; do
for rep in 1 2; do
for v in ${VARS:-old new}; do
  LMKAN_B200_LIB=$PWD/tools/ab/$v/liblmkan_b200.so SWEEP_GRAPH=1 SWEEP=tools/sweep_def.json timeout 300 python tools/sweep.py $c 2>&1 | sed "s/^/cfg$c $v /"
done
done
done

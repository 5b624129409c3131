#!/bin/bash
# A/B timing of library builds on one box: tools/ab/<name>/liblmkan_b200.so
for rep in 1 2; do
for v in ${VARS:-A B C D}; do
  LMKAN_B200_LIB=$PWD/tools/ab/$v/liblmkan_b200.so SWEEP=tools/sweep_def.json timeout 300 python tools/sweep.py ${CFG:-2} 2>&1 | sed "s/^/$v /"
done
done

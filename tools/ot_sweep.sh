#!/bin/bash
# Output-tile width (LMKAN_B200_OT) per layer shape, for choose_out_tile.
mkdir -p gpurun_out
for shape in "64 64 8 16384" "64 64 8 262144" "576 64 16 16384" "576 64 16 65536" "576 64 16 262144" \
             "128 64 28 65536" "128 64 28 1048576" "32 32 12 65536" "288 32 16 65536" "1024 64 16 65536" "128 128 28 1048576"; do
  for ot in 64 32 16; do
    LMKAN_B200_OT=$ot timeout 120 python tools/ubench_shape.py $shape
  done
done

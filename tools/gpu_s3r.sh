set -x
O=gpurun_out/s3r; mkdir -p $O
SWEEP_GRAPH=1 SWEEP='[{}, {"LMKAN_B200_OT":"32"}, {"LMKAN_B200_OT":"16"}, {"LMKAN_B200_OT":"16","LMKAN_B200_MODE":"fused"}, {"LMKAN_B200_OT":"32","LMKAN_B200_MODE":"fused"}]' timeout 600 python tools/sweep.py 1 > $O/sweep1.txt 2>&1; cut -c1-330 $O/sweep1.txt

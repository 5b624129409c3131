set -x
O=gpurun_out/s4f; mkdir -p $O
SWEEP_GRAPH=1 SWEEP='[{}, {"LMKAN_B200_MAX_NBUF":"8"}, {"LMKAN_B200_MAX_NBUF":"10"}, {"LMKAN_B200_MAX_NBUF":"8","LMKAN_B200_OT":"32"}, {"LMKAN_B200_MAX_NBUF":"8","LMKAN_B200_NW":"2"}, {"LMKAN_B200_MAX_NBUF":"8","LMKAN_B200_MODE":"fused"}]' timeout 600 python tools/sweep.py 1 > $O/sweep1.txt 2>&1; cut -c1-260 $O/sweep1.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt

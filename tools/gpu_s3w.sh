set -x
O=gpurun_out/s3w; mkdir -p $O
SWEEP='[{}, {"LMKAN_B200_NW":"8","LMKAN_B200_NBUF":"2"}, {"LMKAN_B200_NW":"8","LMKAN_B200_NBUF":"2","LMKAN_B200_MODE":"staged"}]' timeout 600 python tools/sweep.py 4 > $O/sweep4.txt 2>&1; cut -c1-300 $O/sweep4.txt
SWEEP='[{}, {"LMKAN_B200_NW":"8","LMKAN_B200_NBUF":"2"}]' timeout 600 python tools/sweep.py 2 > $O/sweep2.txt 2>&1; cut -c1-300 $O/sweep2.txt
SWEEP='[{}, {"LMKAN_B200_NW":"8","LMKAN_B200_NBUF":"2"}]' timeout 600 python tools/sweep.py 3 > $O/sweep3.txt 2>&1; cut -c1-300 $O/sweep3.txt

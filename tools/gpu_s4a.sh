set -x
O=gpurun_out/s4a; mkdir -p $O
timeout 120 python tools/split_check.py > $O/split.txt 2>&1; cat $O/split.txt | cut -c1-250
SWEEP='[{}, {"LMKAN_B200_MODE":"split"}, {"LMKAN_B200_MODE":"split","LMKAN_B200_NBUF":"2"}, {"LMKAN_B200_MODE":"split","LMKAN_B200_NBUF":"3"}]' timeout 300 python tools/sweep.py 4 > $O/sweep4.txt 2>&1; cut -c1-250 $O/sweep4.txt

set -x
O=gpurun_out/s4h; mkdir -p $O
VARS="old nv" CFGS="4 3" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-60 $O/ab.txt

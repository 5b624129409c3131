set -x
O=gpurun_out/s3t; mkdir -p $O
VARS="old new" CFGS="2 3 1 4" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-60 $O/ab.txt

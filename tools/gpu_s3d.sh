set -x
O=gpurun_out/s3d; mkdir -p $O
VARS="new v4" CFGS="2 1" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cat $O/ab.txt
LMKAN_B200_LIB=$PWD/tools/ab/v4/liblmkan_b200.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > $O/pytest_v4.txt 2>&1; tail -3 $O/pytest_v4.txt

set -x
O=gpurun_out/s3l; mkdir -p $O
VARS="old new" CFGS="3 2 1" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-300 $O/ab.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt

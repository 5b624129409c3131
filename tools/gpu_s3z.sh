set -x
O=gpurun_out/s3z; mkdir -p $O
VARS="old new" CFGS="4 3" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-60 $O/ab.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt

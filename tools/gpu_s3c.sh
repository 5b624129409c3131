set -x
O=gpurun_out/s3c; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 3 -c 1 -o $O/cfg4_gather -f python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu4.log 2>&1
tail -2 $O/ncu4.log

set -x
O=gpurun_out/s3u; mkdir -p $O
VARS="old new" CFGS="3 2" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-60 $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "records" $O/launches_cfg3.csv | tail -4 | awk -F'","' '{print $(NF)}'
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt

set -x
O=gpurun_out/s3s; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,launch__grid_size --clock-control none --csv --log-file $O/launches_cfg1.csv python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "records|fwd_fused" $O/launches_cfg1.csv | tail -6 | awk -F'","' '{print $5" | "$(NF-2)" "$(NF)}' | cut -c1-60,200-

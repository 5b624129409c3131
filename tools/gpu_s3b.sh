set -x
O=gpurun_out/s3b; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
VARS="old new" CFGS="2 1" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 300 python bench.py --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -c 300 $O/bench_cfg2.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/l4.log 2>&1
grep -c fwd_fused $O/launches_cfg4.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 2 -c 1 -o $O/cfg2_gather -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu2.log 2>&1
tail -2 $O/ncu2.log

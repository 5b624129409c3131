set -x
O=gpurun_out/s3j; mkdir -p $O
VARS="old new" CFGS="4" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-120 $O/ab.txt
for c in 4; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2>&1; echo cfg$c; grep -o '"ms_per_step": [0-9.]*' $O/bench_cfg$c.json; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg$c.json; done
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt

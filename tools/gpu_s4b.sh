set -x
O=gpurun_out/s4b; mkdir -p $O
for c in 1 1 3; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2>&1; echo cfg$c; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg$c.json; done
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt

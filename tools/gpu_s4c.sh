set -x
O=gpurun_out/s4c; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "host_pipeline or host_paths or conv_host or empty" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 300 python bench.py --config 1 > $O/bench_cfg1.json 2>&1; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg1.json

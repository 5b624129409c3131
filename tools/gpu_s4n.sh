set -x
O=gpurun_out/s4n; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "lane_runs" > $O/pytest.txt 2>&1; tail -15 $O/pytest.txt

set -x
O=gpurun_out/s4o; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "f64" > $O/pytest.txt 2>&1; tail -15 $O/pytest.txt

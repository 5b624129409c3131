set -x
O=gpurun_out/s4p; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "across_table_layouts" > $O/pytest.txt 2>&1; tail -15 $O/pytest.txt

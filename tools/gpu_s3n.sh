set -x
O=gpurun_out/s3n; mkdir -p $O
SWEEP_SHARD=8 SWEEP='[{}, {"LMKAN_B200_OT":"32"}, {"LMKAN_B200_OT":"32","LMKAN_B200_SLABS":"2"}, {"LMKAN_B200_OT":"32","LMKAN_B200_SLABS":"3"}]' timeout 900 python tools/sweep.py 5 > $O/sweep5.txt 2>&1; cut -c1-330 $O/sweep5.txt
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "global_offsets or variants or small_batch or duplicated" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt

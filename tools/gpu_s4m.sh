set -x
O=gpurun_out/s4m; mkdir -p $O
SWEEP_SHARD=8 SWEEP='[{}, {"LMKAN_B200_PAR":"0"}, {}, {"LMKAN_B200_PAR":"0"}]' timeout 900 python tools/sweep.py 5 > $O/sweep5.txt 2>&1; cut -c1-200 $O/sweep5.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt

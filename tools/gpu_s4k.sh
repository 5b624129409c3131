set -x
O=gpurun_out/s4k; mkdir -p $O
VARS="old new" CFGS="3 2" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-60 $O/ab.txt
for v in old new; do LMKAN_B200_LIB=$PWD/tools/ab/$v/liblmkan_b200.so LMKAN_B200_MODE=staged timeout 300 python bench.py --config 4 --no-cpu-baseline --no-e2e > $O/b4_$v.json 2>&1; echo $v; grep -o '"ms_per_step": [0-9.]*' $O/b4_$v.json; done
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt

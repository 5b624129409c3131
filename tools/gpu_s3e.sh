set -x
O=gpurun_out/s3e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for d in 0 1 0 1; do LMKAN_B200_DUP16=$d timeout 300 python bench.py --config 4 --no-cpu-baseline > $O/bench_cfg4_dup$d.json 2>&1; echo dup$d; grep -o '"ms_per_step": [0-9.]*' $O/bench_cfg4_dup$d.json; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg4_dup$d.json; done
timeout 300 python bench.py --no-cpu-baseline > $O/bench_cfg2.json 2>&1; grep -o '"ms_per_step": [0-9.]*' $O/bench_cfg2.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 3 -c 1 -o $O/cfg4_gather -f python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu4.log 2>&1

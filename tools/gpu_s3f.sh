set -x
O=gpurun_out/s3f; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for c in 4 2 3 1; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2>&1; echo cfg$c; grep -o '"ms_per_step": [0-9.]*' $O/bench_cfg$c.json; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg$c.json; done
for ch in 4 16; do LMKAN_B200_HOST_CHUNKS=$ch timeout 300 python bench.py --config 2 --no-cpu-baseline --steps 10 > $O/bench_cfg2_ch$ch.json 2>&1; echo ch$ch; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg2_ch$ch.json; done
for cr in 256 1024; do LMKAN_B200_CONV_CHUNK_ROWS=$cr timeout 300 python bench.py --config 4 --no-cpu-baseline > $O/bench_cfg4_cr$cr.json 2>&1; echo cr$cr; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg4_cr$cr.json; done

set -x
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3/pytest.txt 2>&1; tail -3 gpurun_out/s3/pytest.txt
timeout 300 python bench.py > gpurun_out/s3/bench_cfg2.json 2> gpurun_out/s3/bench_cfg2.err; tail -c 600 gpurun_out/s3/bench_cfg2.json
timeout 300 python bench.py --config 4 --no-cpu-baseline > gpurun_out/s3/bench_cfg4.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 6 -c 1 -o gpurun_out/s3/cfg4_gather -f python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3/ncu4.log 2>&1
tail -3 gpurun_out/s3/ncu4.log

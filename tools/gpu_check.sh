#!/bin/bash
# One GPU session: parity tests, a short bench, the ncu launch list and one
# full ncu capture of the fused kernel. Outputs land in gpurun_out/$TAG*.
TAG=${TAG:-r}
CFG=${CFG:-2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/${TAG}_gpu.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.txt 2>&1
  tail -5 gpurun_out/${TAG}_pytest.txt
fi
timeout 600 python bench.py --config $CFG --steps ${STEPS:-20} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 1500 gpurun_out/${TAG}_bench.json
if [ "${NCU:-1}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s ${NCU_SKIP:-3} -c 1 \
     -o gpurun_out/${TAG}_prof -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
  tail -3 gpurun_out/${TAG}_ncu.log
fi

#!/bin/bash
# One ncu --set full capture of the dominant gather kernel of a bench config,
# plus its launch list (per-kernel durations, cold, serialized):
#   TAG=r2_cfg4 CFG=4 KREGEX=fwd_fused SKIP=3 BENCH_ARGS="" bash tools/ncu_capture.sh
# -> gpurun_out/$TAG.ncu-rep, gpurun_out/${TAG}_launches.csv
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-fwd_fused} -s ${SKIP:-3} -c 1 \
    -f -o gpurun_out/$TAG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS \
    > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log

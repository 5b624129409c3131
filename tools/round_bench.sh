#!/bin/bash
# One GPU box: bench lines for every BASELINE config, the reference arm at
# cfg2, the ncu launch list of the default bench command and one --set full
# capture of the cfg2 gather kernel. Outputs under gpurun_out/round/.
set -x
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 400 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
for c in 1 3 4; do timeout 400 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 600 python bench.py --config 5 --shards 8 --steps 5 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_cfg2.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 6 -c 1 -o $O/cfg2_gather python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $O

#!/bin/bash
# One GPU box: ncu launch lists and --set full captures of the dominant gather
# kernels (cfg2, cfg3 layer 2, cfg4) first, folded into profiles/ncu_summary.json
# on the box so the bench lines below report this build's DRAM traffic; then
# bench lines for every BASELINE config and the reference arm at cfg2.
# Outputs under gpurun_out/round/ (tools/update_profiles.py copies them into
# profiles/).
set -x
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 4 -c 1 -f -o $O/cfg2_gather python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 3 -c 1 -f -o $O/cfg4_gather python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 7 -c 1 -f -o $O/cfg3_layer2_gather python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/update_profiles.py --ncu-only
timeout 400 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
for c in 1 3 4; do timeout 400 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 600 python bench.py --config 5 --shards 8 --steps 5 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_cfg2.json 2> $O/bench_ref.err
ls -la $O

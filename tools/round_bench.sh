#!/bin/bash
# One GPU box, end of a round: ncu launch lists and --set full captures of the
# dominant gather kernel of every config (folded into profiles/ncu_summary.json
# on the box so the bench lines below report this build's DRAM traffic), then
# bench lines for every BASELINE config, the reference-precision layer, the
# reference arm and the backward timings. Outputs under gpurun_out/round_$R/;
# `python tools/update_profiles.py` copies them into profiles/ as ${R}_*.
#   R=r2 gpurun -- bash tools/round_bench.sh
R=${R:-r2}
O=gpurun_out/round_$R
mkdir -p $O
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
for c in 1 2 3 4 6 7; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
  python bench.py --config 5 --shards 8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cap() {  # cap <name> <config> <skip> [bench args]
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-fwd_fused} -s $3 -c 1 -f \
    -o $O/$1 python bench.py --config $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${@:4} > /dev/null 2>&1
}
cap cfg2_gather 2 3
cap cfg4_gather 4 3
cap cfg3_layer2_gather 3 7
KREGEX=narrow cap cfg3_head 3 3
cap cfg1_gather 1 3
cap cfg5_gather 5 3 --shards 8
cap cfg6_gather 6 3
cap cfg7_gather 7 3
python tools/update_profiles.py --ncu-only
# the .ncu-rep files are too large to come back (gpurun merges <= 64 MiB):
# keep their extracted key metrics / details and the traffic summary
mkdir -p $O/prof
cp profiles/${R}_*ncu* profiles/ncu_summary.json $O/prof/ 2>/dev/null
rm -f $O/*.ncu-rep
timeout 400 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
for c in 1 3 4 6 7; do timeout 400 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 python bench.py --config 5 --shards 8 --steps 5 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python bench.py --precision 64 --no-cpu-baseline > $O/bench_cfg2_exact.json 2> $O/bench_cfg2_exact.err
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg2.json 2> $O/bench_ref.err
for c in 1 3 4 6 7; do timeout 600 python bench.py --impl reference --config $c > $O/bench_reference_cfg$c.json 2>> $O/bench_ref.err; done
timeout 600 python tools/bench_backward.py > $O/bwd.jsonl 2> $O/bwd.err
ls -la $O

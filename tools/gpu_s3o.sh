set -x
O=gpurun_out/round; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_fused -s 7 -c 1 -f -o $O/cfg3_layer2_gather python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/update_profiles.py --ncu-only
timeout 400 python bench.py --config 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; tail -c 400 $O/bench_cfg3.json
SWEEP='[{}, {"LMKAN_B200_RT":"8"}, {"LMKAN_B200_MODE":"staged"}, {"LMKAN_B200_MODE":"staged","LMKAN_B200_RT":"8"}, {"LMKAN_B200_NBUF":"2"}]' timeout 600 python tools/sweep.py 4 > gpurun_out/sweep4.txt 2>&1; cut -c1-300 gpurun_out/sweep4.txt

set -x
O=gpurun_out/s3x; mkdir -p $O
LMKAN_B200_MODE=staged timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4_staged.csv python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "records|fwd_fused" $O/launches_cfg4_staged.csv | tail -4 | awk -F'","' '{print substr($5,1,40)" "$(NF)}'
LMKAN_B200_MODE=staged timeout 600 ncu --set full --clock-control none --import-source on -k regex:records -s 3 -c 1 -f -o $O/cfg4_k1 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:narrow -s 3 -c 1 -f -o $O/cfg3_head python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $O

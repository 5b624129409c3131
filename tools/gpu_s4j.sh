set -x
O=gpurun_out/s4j; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:records4 -s 7 -c 1 -f -o $O/cfg3_layer2_records python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:narrow -s 3 -c 1 -f -o $O/cfg3_head python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $O

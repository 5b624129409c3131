set -x
O=gpurun_out/s4l; mkdir -p $O
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > $O/mem0.txt; cat $O/mem0.txt
( for i in $(seq 1 60); do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> $O/mem_trace.txt; sleep 5; done ) &
MON=$!
timeout 900 python bench.py --config 5 --shards 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg5_full.json 2> $O/bench_cfg5_full.err
echo rc=$?
kill $MON 2>/dev/null
tail -c 1500 $O/bench_cfg5_full.json; tail -5 $O/bench_cfg5_full.err; sort -n $O/mem_trace.txt | tail -1

mkdir -p gpurun_out
for c in 1 4 6 7; do timeout 600 python bench.py --config $c > gpurun_out/b_cfg$c.json 2> gpurun_out/b_cfg$c.err; done
timeout 300 python bench.py --config 6 --impl reference --steps 3 --warmup 3 > gpurun_out/b_ref6.json 2>&1
timeout 300 python bench.py --config 7 --impl reference --steps 3 --warmup 3 > gpurun_out/b_ref7.json 2>&1

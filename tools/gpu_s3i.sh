set -x
O=gpurun_out/s3i; mkdir -p $O
for t in 0 1 0 1; do LMKAN_B200_HOST_TAPER=$t timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 10 > $O/bench_cfg4_t$t.json 2>&1; echo cfg4 t$t; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg4_t$t.json; done
for t in 0 1 0 1; do LMKAN_B200_HOST_TAPER=$t timeout 300 python bench.py --config 2 --no-cpu-baseline --steps 10 > $O/bench_cfg2_t$t.json 2>&1; echo cfg2 t$t; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg2_t$t.json; done
SWEEP='[{"LMKAN_B200_OT":"64"},{"LMKAN_B200_OT":"32"},{"LMKAN_B200_OT":"32","LMKAN_B200_NBUF":"3"},{"LMKAN_B200_OT":"32","LMKAN_B200_NBUF":"4"},{"LMKAN_B200_OT":"64"}]' timeout 600 python tools/sweep.py 2 > $O/sweep2.txt 2>&1; cut -c1-200 $O/sweep2.txt

set -x
O=gpurun_out/s3y; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
SWEEP='[{}, {"LMKAN_B200_K1":"1"}, {}, {"LMKAN_B200_K1":"1"}]' timeout 600 python tools/sweep.py 3 > $O/sweep3.txt 2>&1; cut -c1-90 $O/sweep3.txt
SWEEP='[{}, {"LMKAN_B200_K1":"1"}, {}, {"LMKAN_B200_K1":"1"}]' timeout 600 python tools/sweep.py 2 > $O/sweep2.txt 2>&1; cut -c1-90 $O/sweep2.txt
VARS="old new" CFGS="3" timeout 900 bash tools/ab_run.sh > $O/ab.txt 2>&1; cut -c1-60 $O/ab.txt
for m in fused staged; do for k in 4 1; do LMKAN_B200_MODE=$m LMKAN_B200_K1=$k timeout 300 python bench.py --config 4 --no-cpu-baseline --no-e2e > $O/b4_${m}_$k.json 2>&1; echo $m $k; grep -o '"ms_per_step": [0-9.]*' $O/b4_${m}_$k.json; done; done
LMKAN_B200_MODE=staged timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4_staged.csv python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "records|fwd_fused" $O/launches_cfg4_staged.csv | tail -4 | awk -F'","' '{print substr($5,1,50)" "$(NF)}'

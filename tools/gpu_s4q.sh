set -x
O=gpurun_out/s4q; mkdir -p $O
for ch in 4 8 6 2 4 8; do LMKAN_B200_MODEL_CHUNKS=$ch timeout 300 python bench.py --config 3 --no-cpu-baseline --steps 10 > $O/b3_$ch.json 2>&1; echo ch$ch; grep -o '"e2e": {"value": [0-9.e+]*' $O/b3_$ch.json; done

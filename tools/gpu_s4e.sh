set -x
O=gpurun_out/s4e; mkdir -p $O
for ch in 8 5 6 10 12 8; do LMKAN_B200_HOST_CHUNKS=$ch timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b_ch$ch.json 2>&1; echo ch$ch; grep -o '"e2e": {"value": [0-9.e+]*' $O/b_ch$ch.json; done

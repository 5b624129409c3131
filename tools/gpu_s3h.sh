set -x
O=gpurun_out/s3h; mkdir -p $O
python tools/pcie_bw.py > $O/pcie.json 2>&1; cat $O/pcie.json
for cr in 128 256 1024 2048; do LMKAN_B200_CONV_CHUNK_ROWS=$cr timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 10 > $O/bench_cfg4_cr$cr.json 2>&1; echo cr$cr; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg4_cr$cr.json; done
for ch in 4 6 12 16; do LMKAN_B200_HOST_CHUNKS=$ch timeout 300 python bench.py --config 2 --no-cpu-baseline --steps 10 > $O/bench_cfg2_ch$ch.json 2>&1; echo ch$ch; grep -o '"e2e": {"value": [0-9.e+]*' $O/bench_cfg2_ch$ch.json; done

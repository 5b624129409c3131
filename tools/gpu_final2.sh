set -x
O=gpurun_out/final2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 700 $O/bench.json
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
python -c "
import numpy as np, threading, paper_2509_07103_b200 as pkg
lay = pkg.Layer.random(64, 64, 8, seed=1)
def work():
    for _ in range(3): lay.forward_host(np.random.rand(5000, 64).astype(np.float32))
ts=[threading.Thread(target=work) for _ in range(4)]
[t.start() for t in ts]; [t.join() for t in ts]
print(\"threads ok\")
"; echo exit=$?

#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_coloring.py -m "gpu" -x -q > $O/r2am_pytest.log 2>&1; echo "rc=$?" >> $O/r2am_pytest.log
cat > /tmp/colt.py <<'PY'
import sys, time, json, os
sys.path.insert(0, '.')
import torch
from paper_1805_10904_b200 import Louvain, inputs
for w in ("rmat24", "sbm"):
    r = inputs.make(w)
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        with Louvain(r.n, r.src, r.dst, r.w, coloring=True) as g:
            g.run()
            q = g.modularity(-1)
            info = [(g.level_stats(l)[0], g.level_colors(l), round(g.level_stats(l)[1]["init"], 1)) for l in range(g.num_levels)]
        torch.cuda.synchronize()
        print(w, rep, round((time.perf_counter() - t) * 1e3, 1), q, info, flush=True)
PY
python /tmp/colt.py > $O/r2am_coop.txt 2>&1
LV_JP_STREAM=1 python /tmp/colt.py > $O/r2am_stream.txt 2>&1
echo done

"""GPU probe: device properties, host info, and a first timing of the C4 path."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

out = {}
p = torch.cuda.get_device_properties(0)
out["device"] = dict(name=p.name, sms=p.multi_processor_count, mem_gb=p.total_memory / 2**30,
                     l2_mb=getattr(p, "L2_cache_size", 0) / 2**20)
out["nproc"] = os.cpu_count()
try:
    out["cpu"] = subprocess.run("lscpu | grep 'Model name'", shell=True, capture_output=True, text=True).stdout.strip()
    out["mem"] = subprocess.run("free -g | head -2", shell=True, capture_output=True, text=True).stdout.strip()
except Exception:
    pass
print(json.dumps(out), flush=True)

for name, mk in [("rmat20", lambda: inputs.rmat(20, 16, seed=4)), ("rmat24", lambda: inputs.rmat(24, 16, seed=4))]:
    t = time.time()
    r = mk()
    tg = time.time() - t
    t = time.time()
    lv = Louvain(r.n, r.src, r.dst, r.w)
    torch.cuda.synchronize()
    tc = time.time() - t
    ts = lv.time_sweeps(3, 5)
    t = time.time()
    lv.run()
    tr = time.time() - t
    st = [lv.level_stats(l) for l in range(lv.num_levels)]
    print(json.dumps(dict(graph=name, gen_s=tg, create_s=tc, run_s=tr, q=lv.modularity(), levels=lv.num_levels,
                          stats=st, run_stats=lv.run_stats(), sweep=ts)), flush=True)
    lv.close()

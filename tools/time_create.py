"""Times louvain_create (CSR build from device-resident COO) for a workload."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10904_b200 import Louvain, inputs
w = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
r = inputs.make(w)
s, d = torch.from_numpy(r.src).cuda(), torch.from_numpy(r.dst).cuda()
wt = None if r.w is None else torch.from_numpy(r.w).cuda()
out = []
for ta in (True, False):
    for i in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        lv = Louvain(r.n, s, d, wt, torch_allocator=ta)
        torch.cuda.synchronize(); out.append((ta, round((time.perf_counter() - t) * 1e3, 1)))
        lv.close()
print(json.dumps({"workload": w, "create_ms(torch_alloc, ms)": out}))

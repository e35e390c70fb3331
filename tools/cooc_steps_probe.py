import os, sys, time, json
sys.path.insert(0, '.')
import torch
from paper_1805_10904_b200 import Louvain, inputs
r = inputs.make("cooc")
dev = torch.device("cuda", 0)
src_d = torch.from_numpy(r.src).to(dev); dst_d = torch.from_numpy(r.dst).to(dev)
s = torch.cuda.Stream(dev); torch.cuda.synchronize(); torch.cuda.set_stream(s)
for rep in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    lv = Louvain(r.n, src_d, dst_d, None, device=0, stream=s, torch_allocator=os.environ.get('TA', '1') == '1')
    t1 = time.perf_counter(); lv.run(); t2 = time.perf_counter()
    st = [lv.level_stats(l)[1] for l in range(lv.num_levels)]
    lv.close(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(rep, "total %.1f create" % ((t3-t0)*1e3), "create %.1f run %.1f close %.1f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3), json.dumps(st)[:200], flush=True)

"""C5 (R-MAT scale 27) on one GPU: create + run from host buffers; reports memory use."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10904_b200 import Louvain, inputs
t = time.time(); r = inputs.rmat(27, 16, seed=5); tg = time.time() - t
alloc = os.environ.get("TORCH_ALLOC", "1") == "1"
t = time.time(); lv = Louvain(r.n, r.src, r.dst, r.w, torch_allocator=alloc); torch.cuda.synchronize(); tc = time.time() - t
print(json.dumps(dict(gen_s=tg, create_s=tc, nnz=lv.nnz(), mem_reserved=torch.cuda.memory_reserved())), flush=True)
t = time.time(); lv.run(); tr = time.time() - t
print(json.dumps(dict(run_s=tr, q=lv.modularity(), levels=lv.num_levels, stats=[lv.level_stats(l) for l in range(lv.num_levels)],
                      run_stats=lv.run_stats())), flush=True)

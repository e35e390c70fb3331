"""Host wall time of each phase of the bench's device-input step (create / run /
partition / close), step by step, to find stalls outside the kernels.

    TA=1 python tools/steps_probe.py sbm      # library memory from torch's caching allocator
    TA=0 python tools/steps_probe.py sbm      # the library's stream-ordered pool
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "sbm"
r = inputs.make(w)
dev = torch.device("cuda", 0)
src_d = torch.from_numpy(r.src).to(dev)
dst_d = torch.from_numpy(r.dst).to(dev)
w_d = None if r.w is None else torch.from_numpy(r.w).to(dev)
out_d = torch.empty(r.n, dtype=torch.int32, device=dev)
s = torch.cuda.Stream(dev)
torch.cuda.synchronize()
torch.cuda.set_stream(s)
ta = os.environ.get("TA", "1") == "1"
for rep in range(10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    lv = Louvain(r.n, src_d, dst_d, w_d, device=0, stream=s, torch_allocator=ta)
    t1 = time.perf_counter()
    lv.run()
    t2 = time.perf_counter()
    lv.partition(-1, out=out_d)
    t3 = time.perf_counter()
    lv.close()
    t4 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(rep, f"wall {(t5 - t0) * 1e3:.1f} events {e0.elapsed_time(e1):.1f} | create {(t1 - t0) * 1e3:.1f} "
          f"run {(t2 - t1) * 1e3:.1f} part {(t3 - t2) * 1e3:.1f} close {(t4 - t3) * 1e3:.1f} "
          f"tail-sync {(t5 - t4) * 1e3:.1f} ms", flush=True)

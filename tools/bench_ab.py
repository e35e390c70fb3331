"""A/B timing of one bench step under different binding options (not a bench value).

    python tools/bench_ab.py [--workload rmat24] [--reps 2]

Variants: torch allocator vs library cudaMallocAsync, torch current stream vs a
dedicated stream vs the library stream, profiling on/off.  Prints ms per step and the
level-0 phase times of each.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_10904_b200 import Louvain, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="rmat24")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
r = inputs.make(args.workload)
dev = torch.device("cuda", 0)
src_d = torch.from_numpy(r.src).to(dev)
dst_d = torch.from_numpy(r.dst).to(dev)
w_d = None if r.w is None else torch.from_numpy(r.w).to(dev)
side = torch.cuda.Stream(dev)
VARIANTS = {
    "torchalloc_curstream_prof": dict(stream="cur", torch_allocator=True, profile=True),
    "torchalloc_curstream": dict(stream="cur", torch_allocator=True, profile=False),
    "torchalloc_ownstream": dict(stream="side", torch_allocator=True, profile=False),
    "mallocasync_libstream": dict(stream=None, torch_allocator=False, profile=False),
    "torchalloc_libstream": dict(stream=None, torch_allocator=True, profile=False),
    "mallocasync_libstream_prof": dict(stream=None, torch_allocator=False, profile=True),
}
out = {}
for name, v in VARIANTS.items():
    st = {"cur": torch.cuda.current_stream(dev), "side": side, None: None}[v["stream"]]
    ts = []
    for rep in range(args.reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lv = Louvain(r.n, src_d, dst_d, w_d, device=0, stream=st, torch_allocator=v["torch_allocator"],
                     profile=v["profile"])
        lv.run()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        phases = lv.level_stats(0)[1]
        lv.close()
        if rep:
            ts.append(dt)
    out[name] = {"ms": sum(ts) / len(ts), "phases_l0": phases}
    print(name, json.dumps(out[name]), flush=True)

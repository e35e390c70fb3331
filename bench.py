#!/usr/bin/env python
"""Benchmark of the GPU Louvain hot path (arXiv 1805.10904) — one JSON line on rank 0.

A *step* is one pass of the whole hot path over one synthetic graph: louvain_create
(CSR build from device-resident COO records) + louvain_run (every level: sweeps,
commit, Q, merge, renumber, contraction) + the final composed partition into a
device buffer.  value = directed-edge visits of all local-move sweeps of the step /
step time (edges/s, whole job over all ranks).  e2e = the same through the public API
from pinned HOST buffers (H2D of the records and D2H of the final partition inside the
timed region).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                        [--impl {native,reference}]
Workloads (BASELINE.json configs): karate, sbm, cooc, rmat24 (default), rmat27.
Inputs are larger than L2 for every workload except karate/sbm (noted in config).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "local-move edges/sec and end-to-end Louvain time at 1/2/4/8 B200; final Q"
UNIT = "edges/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}

# CPU baseline (SURVEY §8(d) "oracle timing: same run, same CSR bytes"): the oracle as it
# stands builds its own CSR of the SAME workload (same seeded records) and runs the first
# sweeps of Algorithm 1 at level 0 — a bounded sample of the same step (the whole run
# would take minutes), timed on 1 core and on every host core (bit-identical results).
# rmat27 (C5) needs ~120 GB of host memory for the oracle's CSR: it keeps a same-recipe
# R-MAT scale-24 sample instead (same_config false).
CPU_SWEEPS_1CORE = 1
CPU_SWEEPS_ALL = 3
REF_SWEEPS = 2  # --impl reference: sweeps per step (Algorithm 1 at level 0, all cores)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return dict(PEAKS_FALLBACK)


def make_workload(name):
    from paper_1805_10904_b200 import inputs

    return inputs.make(name)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("BENCH_CLOCK_MS", "200")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.rows.append(f)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        loaded = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit() and r[6].isdigit() and int(r[6]) > 0]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(loaded or sm) if (loaded or sm) else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def dist_init():
    from paper_1805_10904_b200 import dist as lvd

    rank, world, local = lvd.env_rank()
    if world > 1:
        import torch

        torch.cuda.set_device(local)
        lvd.init_process_group("nccl")
    return world, rank, local


def allmax(x, world):
    from paper_1805_10904_b200 import dist as lvd

    return lvd.allmax(x, device="cuda") if world > 1 else x


def barrier(world):
    from paper_1805_10904_b200 import dist as lvd

    lvd.barrier()


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_ORACLE_G = {}


def oracle_graph(workload, records=None):
    """The oracle's own CSR of the workload (built from the seeded records, never from
    the CUDA path), cached per process; returns (graph, build seconds, description)."""
    import oracle
    from paper_1805_10904_b200 import inputs

    if workload not in _ORACLE_G:
        same = workload != "rmat27"
        r = records if (same and records is not None) else (inputs.make(workload) if same else inputs.rmat(24, 16, seed=5))
        oracle.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        g = oracle.Graph.from_edges(r.n, r.src, r.dst, r.w)
        dt = time.perf_counter() - t0
        desc = workload if same else "R-MAT scale 24 of the C5 recipe (seed 5)"
        _ORACLE_G[workload] = (g, dt, desc, same)
    return _ORACLE_G[workload]


def oracle_sweeps(g, threads, sweeps):
    """Algorithm 1 at level 0, capped at `sweeps` sweeps (+ merge, renumber, Q)."""
    import oracle

    oracle.set_threads(threads)
    t0 = time.perf_counter()
    res = oracle.run(g, max_sweeps=sweeps, max_levels=1)
    dt = time.perf_counter() - t0
    oracle.set_threads(os.cpu_count() or 1)
    return res.edge_visits, dt


def cpu_baseline(workload, records=None):
    """The oracle as it stands, on the same workload's CSR, 1 core and all host cores."""
    g, tb, desc, same = oracle_graph(workload, records)
    ncore = os.cpu_count() or 1
    v1, t1 = oracle_sweeps(g, 1, CPU_SWEEPS_1CORE)
    va, ta = oracle_sweeps(g, ncore, CPU_SWEEPS_ALL)
    return {"value": va / ta, "unit": UNIT, "cores": ncore, "kind": "oracle",
            "sample": f"oracle (OpenMP over the Jacobi sweep, {ncore} threads) on {desc} "
                      f"(n={g.n}, nnz={g.nnz}, the oracle's own CSR of the same records): level-0 Algorithm 1 "
                      f"capped at {CPU_SWEEPS_ALL} sweeps (+merge, renumber, Q) = {va} edge visits in {ta:.2f} s",
            "same_config": same,
            "single_core": {"value": v1 / t1, "unit": UNIT, "cores": 1,
                            "sample": f"same, 1 thread, {CPU_SWEEPS_1CORE} sweep(s): {v1} edge visits in {t1:.2f} s"},
            "oracle_csr_build_s": round(tb, 2), "cpu_model": cpu_model(), "nproc": ncore}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (all host cores) on the same workload;
    each step = Algorithm 1 at level 0 capped at REF_SWEEPS sweeps on the oracle's CSR
    (built once, untimed, from the same seeded records)."""
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    g, tb, desc, same = oracle_graph(args.workload)
    ncore = os.cpu_count() or 1
    for _ in range(min(args.warmup, 1)):
        oracle_sweeps(g, ncore, 1)
    times, visits = [], 0
    for _ in range(args.steps):
        v, dt = oracle_sweeps(g, ncore, REF_SWEEPS)
        times.append(dt)
        visits = v
    T = sum(times) / len(times)
    sample = (f"oracle (OpenMP, {ncore} threads) on {desc} (n={g.n}, nnz={g.nnz}): per step level-0 Algorithm 1 "
              f"capped at {REF_SWEEPS} sweeps (+merge, renumber, Q) = {visits} edge visits; CSR built once "
              f"({tb:.1f} s, untimed)")
    line = {"impl": "reference", "metric": METRIC, "value": visits / T, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": T * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "sample": sample, "same_config": same},
            "cpu_baseline": {"value": visits / T, "unit": UNIT, "cores": ncore, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": visits / T, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def spawn_local_ranks(n):
    """`bench.py --gpus N` without a launcher: start N local ranks (one per GPU) with the
    torchrun environment (127.0.0.1 rendezvous), forward rank 0's output, return the
    worst exit code.  Under torchrun (WORLD_SIZE set) this is not used."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    return max(p.wait() for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="rmat24", choices=["karate", "sbm", "cooc", "rmat24", "rmat27"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--dist-check", action="store_true",
                    help="launcher self-test (CPU, gloo): every rank joins, rank 0 prints world and max over ranks")
    ap.add_argument("--library-pool", action="store_true",
                    help="library device memory from its own stream-ordered pool (default: PyTorch's caching allocator)")
    ap.add_argument("--reorder-steps", type=int, default=1,
                    help="steps timed with the F3 degree-class relabel (reported beside the headline)")
    ap.add_argument("--coloring-steps", type=int, default=1,
                    help="timed steps of the colouring-heuristic variant (SURVEY F2, D29); 0 = skip")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_local_ranks(args.gpus)
    if args.dist_check:
        from paper_1805_10904_b200 import dist as lvd

        rank, world, _ = lvd.env_rank()
        if world > 1:
            lvd.init_process_group("gloo")
        mx = lvd.allmax(float(rank), device="cpu")
        lvd.barrier()
        if rank == 0:
            print(json.dumps({"dist_check": True, "n_gpus": world, "allmax_rank": mx, "gpus_arg": args.gpus}), flush=True)
        return 0
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    from paper_1805_10904_b200 import Louvain

    world, rank, local = dist_init()
    if world > torch.cuda.device_count():
        if rank == 0:
            print(json.dumps({"metric": METRIC, "error": f"{world} ranks but {torch.cuda.device_count()} visible GPUs "
                              "(one process per GPU)"}), flush=True)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    r = make_workload(args.workload)
    m = r.m
    # device-resident inputs (value) and pinned host inputs (e2e)
    src_d = torch.from_numpy(r.src).to(dev)
    dst_d = torch.from_numpy(r.dst).to(dev)
    w_d = None if r.w is None else torch.from_numpy(r.w).to(dev)
    src_h = torch.from_numpy(r.src).pin_memory()
    dst_h = torch.from_numpy(r.dst).pin_memory()
    w_h = None if r.w is None else torch.from_numpy(r.w).pin_memory()
    out_d = torch.empty(r.n, dtype=torch.int32, device=dev)
    # a dedicated (non-default) stream for both legs: the legacy default stream
    # serialises against torch's allocator traffic (tools/bench_ab.py: +25 % step time)
    stream = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    torch.cuda.set_stream(stream)
    # device memory of the library: PyTorch's caching allocator by default; --library-pool
    # uses the library's own stream-ordered pool (cudaMallocAsync, release threshold raised)
    alloc = dict(torch_allocator=not args.library_pool)
    shard = {}
    if world > 1:  # sweep-sharded (strong scaling): graph replicated, vertex ranges split
        from paper_1805_10904_b200 import dist as lvd

        comm, _, _ = lvd.nccl_comm(local)
        shard = dict(nccl_comm=comm, rank=rank, world=world)

    def step(profile=False):
        lv = Louvain(r.n, src_d, dst_d, w_d, device=local, stream=stream, profile=profile and world == 1, **shard,
                     **alloc)
        lv.run()
        lv.partition(-1, out=out_d)
        st = lv.run_stats()
        info = dict(nnz=lv.nnz(), edge_visits=st["edge_visits"], launches=st["launches"], q=lv.modularity(-1),
                    levels=lv.num_levels, sweeps=[lv.level_stats(l)[0] for l in range(lv.num_levels)],
                    times=[lv.level_stats(l)[1] for l in range(lv.num_levels)])
        if profile:
            info["profile"] = lv.profile()
        lv.close()
        return info

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    infos = []
    e0.record(stream)
    for _ in range(args.steps):
        infos.append(step())
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms = allmax(ms, world)
    # per-kernel CUDA events (on each kernel's launching stream) cost host time per launch,
    # so they run in one extra step after the timed ones, itself timed for the shares
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    pinfo = step(profile=True)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    visits = infos[-1]["edge_visits"]  # of the whole graph (every rank reports the same)
    value = visits / (ms / 1e3)

    # e2e through the public API from pinned host buffers (H2D + D2H inside the region)
    host_out = np.empty(r.n, dtype=np.int32)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        with Louvain(r.n, src_h.numpy(), dst_h.numpy(), None if w_h is None else w_h.numpy(), device=local,
                     stream=stream, **shard, **alloc) as lv:
            lv.run()
            host_out[:] = lv.partition(-1)
    torch.cuda.synchronize()
    e2e_ms = allmax((time.perf_counter() - t0) * 1e3 / max(args.e2e_steps, 1), world)
    h2d = m * (4 + 4 + (0 if r.w is None else r.w.itemsize))
    d2h = r.n * 4

    # the colouring heuristic (reading D29): same workload, same timing,
    # reported beside the paper's synchronous sweeps (not the headline value)
    coloring = None
    if args.coloring_steps > 0:
        def cstep():
            lv = Louvain(r.n, src_d, dst_d, w_d, device=local, stream=stream, coloring=True, **alloc)
            lv.run()
            lv.partition(-1, out=out_d)
            ci = dict(q=lv.modularity(-1), sweeps=[lv.level_stats(l)[0] for l in range(lv.num_levels)],
                      colors=[lv.level_colors(l)[0] for l in range(lv.num_levels)],
                      visits=lv.run_stats()["edge_visits"],
                      times=[lv.level_stats(l)[1] for l in range(lv.num_levels)])
            lv.close()
            return ci
        if world == 1:
            cstep()
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            for _ in range(args.coloring_steps):
                ci = cstep()
            c1.record(stream)
            torch.cuda.synchronize()
            cms = c0.elapsed_time(c1) / args.coloring_steps
            coloring = {"end_to_end_s": cms / 1e3, "value": ci["visits"] / (cms / 1e3), "unit": UNIT,
                        "final_q": ci["q"], "sweeps_per_level": ci["sweeps"], "colors_per_level": ci["colors"],
                        "color_classes": 32, "init_ms_per_level": [round(t["init"], 1) for t in ci["times"]],
                        "note": "colouring heuristic (D29): colour classes swept in turn; init includes the "
                                "Jones-Plassmann colouring"}

    # F3 degree-class relabel (louvain_config.reorder): same workload and timing,
    # the method on the relabelled graph (a different, equally valid tie-break order), so
    # reported beside the headline, not as it
    reorder = None
    if args.reorder_steps > 0 and world == 1:
        def rstep():
            lv = Louvain(r.n, src_d, dst_d, w_d, device=local, stream=stream, reorder=True, **alloc)
            lv.run()
            lv.partition(-1, out=out_d)
            ri = dict(q=lv.modularity(-1), sweeps=[lv.level_stats(l)[0] for l in range(lv.num_levels)],
                      visits=lv.run_stats()["edge_visits"])
            lv.close()
            return ri
        rstep()
        torch.cuda.synchronize()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(args.reorder_steps):
            ri = rstep()
        q1.record(stream)
        torch.cuda.synchronize()
        rms = q0.elapsed_time(q1) / args.reorder_steps
        reorder = {"end_to_end_s": rms / 1e3, "value": ri["visits"] / (rms / 1e3), "unit": UNIT,
                   "final_q": ri["q"], "sweeps_per_level": ri["sweeps"], "steps": args.reorder_steps,
                   "note": "F3: vertices relabelled by decreasing degree class before the CSR build "
                           "(step time includes the relabel)"}

    # roofline of the dominant kernel over the timed region
    pk = peaks()
    agg = {}
    for inf in [pinfo]:
        for k in inf.get("profile", {"kernels": []})["kernels"]:
            a = agg.setdefault(k["name"], [0.0, 0.0, 0.0])
            a[0] += k["ms"]
            a[1] += k["alg_bytes"]
            a[2] += k["launches"]
    sweep_pass = agg.pop("sweep_pass", None)  # whole-pass wall time (all bins, concurrent)
    top = max(agg, key=lambda k: agg[k][0]) if agg else None
    t_ms, t_bytes, t_launch = agg[top] if agg else (None, None, None)
    achieved = t_bytes / (t_ms / 1e3) / 1e9 if agg else None
    sweep_ms = sweep_pass[0] if sweep_pass else None
    traffic, traffic_note = None, None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):  # DRAM bytes of one ncu --set full capture of this kernel
        try:
            t = json.load(open(tf)).get(args.workload, {}).get(top)
            if t:
                traffic = t["bytes"]
                traffic_note = (f"{t['launch']}; that launch's algorithmic bytes: {t['alg_bytes_same_launch']:.4g} "
                                f"(traffic/algorithmic = {t['bytes'] / t['alg_bytes_same_launch']:.2f})")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"] if agg else None, "traffic": traffic, "traffic_note": traffic_note,
                "kernel": top, "kernel_ms_per_launch": t_ms / t_launch if agg else None,
                "alg_bytes_per_launch": t_bytes / t_launch if agg else None,
                "kernel_share_of_step": t_ms / prof_ms if agg else None, "profiled_step_ms": prof_ms,
                "peak_source": pk["source"],
                "note": "per-kernel times: CUDA events on each kernel's launching stream during one profiled step "
                        "run right after the timed steps (same workload; events cost host time per launch); "
                        "achieved = algorithmic bytes (DESIGN.md §6) / time, averaged over all levels' launches"
                        + ("" if agg else "; the sweep-sharded mode (N > 1) has no per-kernel timer: see the N = 1 line")}
    sweep_roof = None
    if sweep_pass:
        sp_ms, sp_bytes, sp_n = sweep_pass
        sweep_roof = {"achieved": sp_bytes / (sp_ms / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                      "frac": sp_bytes / (sp_ms / 1e3) / 1e9 / pk["hbm_gbs"], "ms_per_sweep": sp_ms / sp_n,
                      "alg_bytes_per_sweep": sp_bytes / sp_n, "sweeps": sp_n}

    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(args.workload, r)
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}
    inf = infos[-1]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "graph": r.name, "n": r.n, "records": m,
                   "allocator": "library stream-ordered pool" if args.library_pool else "torch caching allocator",
                   "directed_edges": inf["nnz"], "edge_visits_per_step": visits, "levels": inf["levels"],
                   "sweeps_per_level": inf["sweeps"], "stop_rule": "alg1_abs", "max_sweeps": 100,
                   "parallelism": f"sweep-shard{world} (graph replicated, NCCL label exchange)" if world > 1
                   else "single",
                   "l2": "inputs larger than L2 (126 MB)" if m * 12 > 126e6 else "inputs fit in L2"},
        "end_to_end_s": ms / 1e3, "final_q": inf["q"],
        "sweep_kernels_ms_per_step": sweep_ms,
        "gpu_launches": inf["launches"],
        "roofline": roofline,
        "sweep_roofline": sweep_roof,
        "cpu_baseline": cpu,
        "e2e": ({"value": visits / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                 "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms} if args.e2e_steps > 0 else None),
        "clocks": clk,
        "coloring": coloring,
        "reorder": reorder,
        "phase_ms_level0": inf["times"][0],
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

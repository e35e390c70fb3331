"""Summarise one GPU round (tools/gpu_round.sh TAG) into profiles/TAG_summary.md and
update profiles/traffic.json with the DRAM bytes of the bench's dominant kernel.

    python tools/summarize_round.py TAG

Inputs (gpurun_out/): TAG_bench.json, TAG_launches.csv (ncu --metrics
gpu__time_duration.sum of one bench step), TAG_sweep_full_raw.csv (ncu --set full of one
level-0 C4 sweep) and TAG_ncu_full.log (the time_sweeps JSON of that capture, with the
algorithmic bytes of each kernel in the captured sweep).
"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
bench = json.load(open(os.path.join(G, f"{tag}_bench.json")))
out = [f"# {tag} — measurement summary (B200, sm_100a)\n",
       "All numbers measured on the pool's B200 through `gpurun`; raw files beside this one.\n"]

r = bench["roofline"]
out.append("## Bench line (`python bench.py`, C4 = R-MAT scale 24, ef 16, weights 1-16)\n")
out.append(f"- value: **{bench['value'] / 1e9:.1f} G local-move edge visits/s**, {bench['ms_per_step']:.0f} ms per "
           f"full multi-level run (sweeps per level {bench['config']['sweeps_per_level']}), final Q "
           f"{bench['final_q']:.4f}; e2e from pinned host buffers {bench['e2e']['value'] / 1e9:.1f} G/s "
           f"({bench['e2e']['ms_per_step']:.0f} ms incl. {bench['e2e']['h2d_bytes_per_step'] / 1e9:.1f} GB H2D)")
out.append(f"- dominant kernel `{r['kernel']}`: {r['achieved']:.0f} GB/s algorithmic = {r['frac']:.3f} of "
           f"{r['peak']:.0f} GB/s ({r['peak_source']}); share of the profiled step {r['kernel_share_of_step']:.3f}")
sr = bench.get("sweep_roofline") or {}
if sr:
    out.append(f"- whole sweep pass (all bins): {sr['achieved']:.0f} GB/s algorithmic = {sr['frac']:.3f} of peak, "
               f"{sr['ms_per_sweep']:.2f} ms per sweep averaged over all levels")
cb = bench.get("cpu_baseline") or {}
if cb.get("value"):
    out.append(f"- CPU oracle (cores {cb['cores']}): {cb['value'] / 1e6:.0f} M edge visits/s — {cb['sample']}")
col = bench.get("coloring")
if col:
    out.append(f"- colouring heuristic (D29): {col['end_to_end_s'] * 1e3:.0f} ms per run, Q {col['final_q']:.4f}, "
               f"sweeps {col['sweeps_per_level']}, colours {col['colors_per_level']}, colouring "
               f"{col['init_ms_per_level']} ms per level")
out.append(f"- clocks: {bench['clocks']}\n")

# launch list of one bench step
lf = os.path.join(G, f"{tag}_launches.csv")
if os.path.exists(lf):
    rows = [x for x in csv.reader(open(lf)) if len(x) > 14 and x[12] == "gpu__time_duration.sum"]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for x in rows:
        name = re.sub(r"\(.*", "", x[4]).replace("void ", "").replace("lv::", "")
        v = float(x[14]) / (1e6 if x[13] == "ns" else 1e3 if x[13] == "us" else 1)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out.append(f"## Launches of `bench.py --steps 1 --warmup 0` (the timed step + the profiled step; `{tag}_launches.csv`: ncu --metrics gpu__time_duration.sum "
               f"--clock-control none; cold-cache, serialised)\n")
    out.append(f"{len(rows)} launches, total kernel time {T:.1f} ms.\n")
    out.append("| share | total ms | launches | kernel |\n|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k])[:20]:
        out.append(f"| {tot[k] / T:.1%} | {tot[k]:.2f} | {cnt[k]} | `{k}` |")
    out.append("")

# ncu --set full of one level-0 sweep
rf = os.path.join(G, f"{tag}_sweep_full_raw.csv")
alg = {}
lg = os.path.join(G, f"{tag}_ncu_full.log")
if os.path.exists(lg):
    m = re.search(r"(\{\"ms_sweep.*\})", open(lg).read())
    if m:
        for k in json.loads(m.group(1))["kernels"]:
            alg[k["name"]] = k["alg_bytes"]
NAME2BIN = {"k_agg_smem<1024": "sweep:agg_blk1024_c16384", "k_agg_smem<512": "sweep:agg_blk512_c8192",
            "k_agg_smem<256": "sweep:agg_blk256_c4096", "k_agg_smem<128": "sweep:agg_blk128_c1024",
            "k_agg_smem<32": "sweep:agg_g32_c256", "k_agg_reg<32": "sweep:reg_g32", "k_sweep_reg<16": "sweep:reg_g16",
            "k_sweep_reg<8": "sweep:reg_g8", "k_sweep_thr<8": "sweep:reg_g8", "k_sweep_reg<4": "sweep:reg_g4",
            "k_sweep_thr<4": "sweep:reg_g4", "k_hub_acc": "sweep:hub_acc", "k_hub_fin": "sweep:hub_fin",
            "k_hub_decide": "sweep:hub_decide"}
if os.path.exists(rf):
    rows = list(csv.reader(open(rf)))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    out.append(f"## Sweep kernels (`{tag}_ncu_full_sweep_kernels_raw.csv`: ncu --set full, one level-0 C4 sweep "
               "after 3 warm sweeps)\n")
    out.append("| kernel | ms | DRAM read MB | DRAM write MB | algorithmic MB | DRAM GB/s | L2 hit % | warps active % | "
               "regs |\n|---|---|---|---|---|---|---|---|---|")
    traffic = json.load(open(os.path.join(P, "traffic.json"))) if os.path.exists(os.path.join(P, "traffic.json")) else {}
    for d in data:
        name = d[ix["Kernel Name"]]
        short = re.sub(r"\(.*", "", name).replace("void ", "").replace("lv::", "")
        ms = float(d[ix["gpu__time_duration.sum"]])
        rd, wr = float(d[ix["dram__bytes_read.sum"]]), float(d[ix["dram__bytes_write.sum"]])
        key = next((v for k, v in NAME2BIN.items() if short.startswith(k)), None)
        a = alg.get(key, 0.0) / 1e6 if key else 0.0
        out.append(f"| `{short}` | {ms:.3f} | {rd:.0f} | {wr:.0f} | {a:.0f} | {(rd + wr) / ms:.0f} | "
                   f"{float(d[ix['lts__t_sector_hit_rate.pct']]):.1f} | "
                   f"{float(d[ix['sm__warps_active.avg.pct_of_peak_sustained_active']]):.1f} | "
                   f"{d[ix['launch__registers_per_thread']]} |")
        if key == r["kernel"] and a > 0:
            traffic.setdefault("rmat24", {})[key] = {
                "bytes": (rd + wr) * 1e6, "alg_bytes_same_launch": a * 1e6,
                "launch": f"level-0 sweep 4 (after 3 warm sweeps) of tools/profile_sweep.py --workload rmat24; "
                          f"ncu --set full --clock-control none ({tag})"}
    json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
    out.append("")
open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))

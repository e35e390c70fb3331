#!/bin/bash
# Per-kernel sweep times (tools/profile_sweep.py, CUDA events) under build/env variants.
# Usage: bash tools/variants.sh "NAME:ENV..." ...   (ENV like LV_SO=... LV_REG_WAVES4=1)
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs python tools/profile_sweep.py --warm 3 --reps 5 > gpurun_out/var_$name.json 2>&1
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/var_{name}.json"))
except Exception as e:
    print(name, "failed", open(f"gpurun_out/var_{name}.json").read()[-300:]); sys.exit()
ks = {k["name"].split(":")[-1]: k["ms"] for k in d["kernels"]}
print(f"{name:14s} sweep {d['ms_sweep']:.3f} ms | " + " ".join(f"{k}={v:.3f}" for k, v in ks.items() if k not in ("sweep_pass",)))
PY
done

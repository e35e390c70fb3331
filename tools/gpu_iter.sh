#!/bin/bash
# One iteration on the B200 box: parity tests (not slow), per-kernel sweep times of
# variants (tools/variants.sh specs in $VARIANTS), and a short bench line.
# Usage: TAG=r2a VARIANTS="old:LV_OLD_SWEEP=1 new:" bash tools/gpu_iter.sh [pytest-args]
TAG=${TAG:-iter}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/${TAG}_smi.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m "gpu and not slow" -x -q "$@" > $O/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> $O/${TAG}_pytest.log
fi
if [ -n "${VARIANTS:-}" ]; then
  bash tools/variants.sh $VARIANTS > $O/${TAG}_variants.txt 2>&1
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
  timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 ${BENCH_ARGS:-} > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
fi
echo done

#!/bin/bash
# A/B of library variants (paper_2502_01826_b200/lib/var/*.so): bench phases, 2 reps each.
# VARS="a b" PYTEST="-k expr" TAG=x bash tools/gpu_ab3.sh
set -u
mkdir -p gpurun_out
TAG=${TAG:-ab}
if [ -n "${PYTEST:-}" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu $PYTEST > gpurun_out/${TAG}_pytest.txt 2>&1
  tail -3 gpurun_out/${TAG}_pytest.txt
fi
for v in ${VARS}; do
  export RFS_LIB_PATH=$PWD/paper_2502_01826_b200/lib/var/$v.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], {k: round(v, 4) for k, v in d['phase_ms'].items()})"
  done
done

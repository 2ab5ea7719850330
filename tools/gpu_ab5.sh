#!/bin/bash
# A/B of library variants on value + e2e (graph replays), two reps each
set -u
mkdir -p gpurun_out
TAG=${TAG:-ab5}
for v in ${VARS}; do
  export RFS_LIB_PATH=$PWD/paper_2502_01826_b200/lib/var/$v.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['ms_per_step'], {k: round(v, 4) for k, v in d['phase_ms'].items() if k in ('bwd_gauss','backward_rays','grad_geom')})"
  done
done

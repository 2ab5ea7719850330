#!/bin/bash
# A/B of library variants: graph-replay value + eager phases + per-kernel ncu time of KRE
set -u
mkdir -p gpurun_out
TAG=${TAG:-ab4}
for v in ${VARS}; do
  export RFS_LIB_PATH=$PWD/paper_2502_01826_b200/lib/var/$v.so
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${v}_l.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --eager > /dev/null 2>&1
  echo "$v $(grep -E "${KRE}" gpurun_out/${TAG}_${v}_l.csv | tail -1 | awk -F'","' '{print $NF}')"
  for rep in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['config']['graph']['eager_ms_per_step'], {k: round(v, 4) for k, v in d['phase_ms'].items() if k in ('bwd_gauss','backward_rays','grad_geom')})"
  done
done

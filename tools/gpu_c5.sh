#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-c5}
for m in "--graph" ""; do
  RFS_DEBUG_STATS=1 timeout 900 python tools/bench_density.py --iterations ${ITERS:-600} $m > gpurun_out/${TAG}${m}.json 2> gpurun_out/${TAG}${m}.err
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}${m}.json')); print('$m', {k:d[k] for k in ('ms_per_iteration_plain','ms_per_iteration_whole_run','ms_median_by_50','loop_counts','n_end')})"
done

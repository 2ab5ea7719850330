#!/bin/bash
# K6 A/B over RFS_HITS_LPR (1: k_hits, 2: k_hits2 CH 32, 3: k_hits2 CH 16): parity, kernel time, bench
mkdir -p gpurun_out
TAG=${TAG:-hab}
for L in ${LPRS:-1 2 3}; do
  RFS_HITS_LPR=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -m gpu -x > gpurun_out/${TAG}_L${L}_tests.txt 2>&1
  echo "L$L tests rc=$? $(tail -1 gpurun_out/${TAG}_L${L}_tests.txt)"
  RFS_HITS_LPR=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_L${L}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --eager > /dev/null 2>&1
  grep "k_hits" gpurun_out/${TAG}_L${L}_launches.csv | awk -F'","' '{print $5, $NF}' | tail -1 | cut -c1-40,200-
  RFS_HITS_LPR=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${TAG}_L${L}_bench.json 2>/dev/null
  python -c "
import json
b=json.loads(open('gpurun_out/${TAG}_L${L}_bench.json').read().strip().splitlines()[-1]); print('L$L', b['value'], b['e2e']['value'], b['config'].get('graph'))"
done

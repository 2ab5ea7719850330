# K6 work: parity + per-warp timing + bench for the given split thresholds
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q ${PYK:-} > gpurun_out/split_pytest.txt 2>&1
tail -3 gpurun_out/split_pytest.txt
for sm in ${SPLITS:-0}; do
  timeout 200 python tools/k6_timing.py 100000 $sm 2>&1
  RFS_K6_SPLIT=$sm timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/split_${sm}.json 2> gpurun_out/split_${sm}.err
  python -c "
import json; d=json.loads(open('gpurun_out/split_${sm}.json').read().strip().splitlines()[-1]); print('split', ${sm}, d['value'], d['ms_per_step'], d['phase_ms'])"
done

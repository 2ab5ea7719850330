# A/B of library variants in paper_2502_01826_b200/lib/var/*.so: K6 per-warp timing + bench phases
set -u
mkdir -p gpurun_out
if [ -n "${PYK:-}" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$PYK" > gpurun_out/ab_pytest.txt 2>&1
  tail -3 gpurun_out/ab_pytest.txt
fi
for v in ${VARS:-a b}; do
  export RFS_LIB_PATH=$PWD/paper_2502_01826_b200/lib/var/$v.so
  echo "== variant $v"
  timeout 200 python tools/k6_timing.py 100000 2>&1 | grep -v "list length\|q0"
  for rep in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['phase_ms'])"
  done
done

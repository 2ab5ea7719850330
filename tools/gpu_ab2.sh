# A/B of library variants (lib/var/<v>.so): bench step time + per-kernel launch list of each
set -u
mkdir -p gpurun_out
for v in ${VARS:-o0 o1}; do
  export RFS_LIB_PATH=$PWD/paper_2502_01826_b200/lib/var/$v.so
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab2_$v.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  python tools/launch_list.py gpurun_out/ab2_$v.csv 2>&1 | grep -E "${KRE:-k_bwd_gauss_v|k_grad_tx|k_forward_v}" | sed "s/^/$v /"
done

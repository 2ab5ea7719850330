#!/bin/bash
# launch lists of config 2 (bench step) and config 5 (training iteration) + bench line
mkdir -p gpurun_out
TAG=${TAG:-r2x}
[ -n "$PYTEST" ] && { timeout 1200 python -m pytest $PYTEST -q -m gpu -x > gpurun_out/${TAG}_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.txt; tail -2 gpurun_out/${TAG}_tests.txt; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c5_launches.csv python tools/bench_density.py --iterations 8 --eager --batch 16 > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${TAG}_c5_launches.csv > gpurun_out/${TAG}_c5_launches.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --eager > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt
python tools/bench_density.py --iterations 400 --batch 16 > gpurun_out/${TAG}_density.json 2> gpurun_out/${TAG}_density.err
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo C5; head -${NK:-14} gpurun_out/${TAG}_c5_launches.txt; echo C2; head -${NK:-14} gpurun_out/${TAG}_launches.txt
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_density.json')); print({k:d[k] for k in ('ms_per_iteration_plain','ms_per_iteration_whole_run','loop_counts','loss_last')})
b=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print(b['value'], b['e2e']['value'], b['config'].get('graph'))"

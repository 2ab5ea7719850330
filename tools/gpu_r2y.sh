#!/bin/bash
# FFMA2 round: GPU tests, loss timing + launch list, config-2 launch list, bench
mkdir -p gpurun_out
TAG=${TAG:-r2y}
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.txt
python tools/prof_loss.py > gpurun_out/${TAG}_loss.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_loss_launches.csv python tools/prof_loss.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --eager > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_tests.txt; cat gpurun_out/${TAG}_loss.txt; grep -E "k_ssim|k_loss|k_frame" gpurun_out/${TAG}_loss_launches.csv | awk -F'","' '{print $5, $NF}' | tail -4
head -8 gpurun_out/${TAG}_launches.txt
python -c "
import json
b=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print(b['value'], b['e2e']['value'], b['config'].get('graph'), b['e2e'].get('step'))"

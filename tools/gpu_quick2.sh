# parity tests + bench + launch list (tag $1)
set -u
mkdir -p gpurun_out
T=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
tail -3 gpurun_out/${T}_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json,sys; d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['phase_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt 2>&1
head -30 gpurun_out/${T}_launches.txt

# launch list of one bench step (tag $1)
set -u
mkdir -p gpurun_out
T=${1:-ll}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt 2>&1
head -40 gpurun_out/${T}_launches.txt

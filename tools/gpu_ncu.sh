# launch list + ncu --set full of selected kernels (regex $2), tag $1
set -u
mkdir -p gpurun_out
T=${1:-n}
K=${2:-"k_bwd|k_lam|k_grad_tx|k_forward"}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt 2>&1
cat gpurun_out/${T}_launches.txt | head -40
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"$K" -c ${3:-8} \
    -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
echo done

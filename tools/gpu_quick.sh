# quick GPU check: parity tests + default bench (+ optional extra args for bench)
set -u
mkdir -p gpurun_out
T=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
tail -3 gpurun_out/${T}_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -c 1500 gpurun_out/${T}_bench.json

#!/bin/bash
# captured training iterations: GPU tests of the train loop + config-5 timing, eager vs captured
mkdir -p gpurun_out
TAG=${TAG:-r2t}
[ -n "$NOTEST" ] || python -m pytest tests/test_train.py -q -m gpu -x -k "captured or fits or nonfinite" > gpurun_out/${TAG}_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.txt
for b in ${BATCHES:-16 1}; do
python tools/bench_density.py --iterations 400 --batch $b > gpurun_out/${TAG}_density_graph_b$b.json 2> gpurun_out/${TAG}_density_graph_b$b.err
python tools/bench_density.py --iterations 400 --batch $b --eager > gpurun_out/${TAG}_density_eager_b$b.json 2> gpurun_out/${TAG}_density_eager_b$b.err
done
tail -3 gpurun_out/${TAG}_tests.txt
for f in gpurun_out/${TAG}_density_*.json; do echo $f; python -c "
import json,sys; d=json.load(open('$f')); print({k:d[k] for k in ('batch_tx','ms_per_iteration_plain','ms_per_iteration_whole_run','idle_between_iterations_ms','loop_counts','density_events','loss_last')})"; done

set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --overlap > gpurun_out/s1_bench_ov.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --overlap --index-side > gpurun_out/s1_bench_ov2.json 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --gaussians 1000000 > gpurun_out/s1_bench_1m.json 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --gaussians 500000 > gpurun_out/s1_bench_500k.json 2>&1
echo done

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 --ignore=tests/test_gpu_parity_r2.py > gpurun_out/r2a_gpu_main.log 2>&1; echo "main rc=$?"
tail -30 gpurun_out/r2a_gpu_main.log
timeout 1800 python -m pytest tests/test_gpu_parity_r2.py -m gpu -q --durations=25 > gpurun_out/r2a_gpu_r2.log 2>&1; echo "r2 rc=$?"
tail -40 gpurun_out/r2a_gpu_r2.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/r2a_bench.log

mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/smoke.txt; tail -3 gpurun_out/bench.txt

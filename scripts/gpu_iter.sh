# one build->measure iteration: GPU tests, bench, ncu full profile of the fused kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench.txt 2>&1
if [ "${PROFILE:-1}" = "1" ]; then bash scripts/gpu_ncu.sh ${KREGEX:-stage_fused} 2 2 > /dev/null 2>&1; fi
tail -3 gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/bench.txt | cut -c1-400

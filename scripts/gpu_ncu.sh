mkdir -p gpurun_out
K=${1:-stage_fused}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${2:-2} -c ${3:-2} -o gpurun_out/prof_$K -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extras > gpurun_out/ncu_$K.log 2>&1
tail -3 gpurun_out/ncu_$K.log

# ncu full capture of one stage-1 + stage-2 pair of the fused kernels, FULL vs GATHER fill mode
mkdir -p gpurun_out
for m in 0 1; do
  ORCHA_FILL_MODE=$m timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stage_fused|fill" -s 3 -c 3 \
    -o gpurun_out/prof_mode$m -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extras --no-variants \
    > gpurun_out/ncu_mode$m.log 2>&1
  tail -2 gpurun_out/ncu_mode$m.log
done

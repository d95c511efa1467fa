# launch list (cold, serialised) of a short bench run: per-kernel durations
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -s ${SKIP:-16} -c ${COUNT:-20} --csv \
    --log-file gpurun_out/launches${TAG}.csv python bench.py --steps 5 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-extras --no-variants > gpurun_out/ncu_launches${TAG}.log 2>&1
python scripts/launch_shares.py gpurun_out/launches${TAG}.csv

# Round-2b profile set: full bench line, launch list of the bench command (cold,
# serialised), one ncu --set full capture of the three advance kernels of a
# steady-state step.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16 -c 24 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 4 --e2e-steps 0 --no-cpu-baseline \
    --no-extras --no-variants > gpurun_out/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stage_fused -s 3 -c 3 \
    -o gpurun_out/prof_stage_fused -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    --no-extras --no-variants > gpurun_out/ncu_stage_fused.log 2>&1
tail -c 300 gpurun_out/bench_full.json

# Round profile set (committed under profiles/): launch list of the bench
# command (cold, serialised: compare shares), full ncu captures of the stage
# kernels and the fill, nvidia-smi clocks during a bench run.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16 -c 20 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-extras --no-variants > gpurun_out/ncu_launches.log 2>&1
bash scripts/gpu_ncu.sh stage_fused 2 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fill -s 0 -c 1 -o gpurun_out/prof_fill -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extras --no-variants > gpurun_out/ncu_fill.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.txt 2>&1
tail -1 gpurun_out/bench_full.txt | cut -c1-200

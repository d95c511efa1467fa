# A/B of environment switches on cfg4: each entry of $VARIANTS ("name:VAR=val,VAR2=val")
# benched interleaved REPS times (bench.py --steps 10 --warmup 3, no extras).
mkdir -p gpurun_out
REPS=${REPS:-2}
for r in $(seq $REPS); do
  for v in $VARIANTS; do
    name=${v%%:*}; envs=${v#*:}
    echo "== $name ($envs)" >> gpurun_out/ab.txt
    env $(echo "$envs" | tr ',' ' ') timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extras --no-variants ${BENCH_ARGS} 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('advance_ms'), d['value'])" >> gpurun_out/ab.txt 2>&1
  done
done
cat gpurun_out/ab.txt

# A/B of experiment libraries (exp/*.so, built by `python -m paper_2507_09337_b200.build --experiment`):
# bench each one (and the default build) on cfg4, interleaved, REPS times.
mkdir -p gpurun_out
REPS=${REPS:-2}
for r in $(seq $REPS); do
  for lib in default exp/*.so; do
    if [ "$lib" = default ]; then unset ORCHA_LIB; else export ORCHA_LIB=$PWD/$lib; fi
    echo "== $lib" >> gpurun_out/ab.txt
    timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-extras ${BENCH_ARGS} 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('advance_ms'), d['value'])" >> gpurun_out/ab.txt 2>&1
  done
done
unset ORCHA_LIB
cat gpurun_out/ab.txt

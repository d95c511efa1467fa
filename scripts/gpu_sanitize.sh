# compute-sanitizer over the fused stage kernels and the fill / pack / dt
# kernels on small grids: memcheck, racecheck (shared memory hazards),
# synccheck (barrier misuse).  Summaries -> gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
T="tests/test_gpu_fillmode.py::test_gather_mode_equals_full_mode"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-regex kns=orcha --print-limit 20 \
    python -m pytest -x -q -p no:cacheprovider "$T" -k "nb1 or nb2" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.txt | tail -4
done

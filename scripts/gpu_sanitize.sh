# compute-sanitizer over this library's kernels (fused stage kernels of both
# methods and both schemes, fill / pack / dt / device-dt kernels) on small
# grids: memcheck, racecheck (shared memory hazards), synccheck (barrier
# misuse).  Summaries -> gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
T="tests/test_gpu_fillmode.py::test_gather_mode_equals_full_mode tests/test_gpu_devdt.py::test_device_dt_loop_with_scheme_variants tests/test_gpu_devdt.py::test_cuda_graph_of_device_dt_steps_equals_plain_loop"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-regex kns=orcha --print-limit 20 \
    python -m pytest -x -q -p no:cacheprovider $T -k "nb1 or nb2 or scheme or graph" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.txt | tail -4
done

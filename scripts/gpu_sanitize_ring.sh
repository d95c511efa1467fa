# compute-sanitizer over the borrowed-ring kernels (box / 18 x 18 / interior
# stage 1 with their ring pushes, gather and full-fill flavours, the plain
# stage 2 with register-carried z fluxes, the concurrent side-stream launch):
# memcheck, racecheck (shared memory hazards), synccheck on small grids.
# Summaries -> gpurun_out/sanitize_ring_*.txt
mkdir -p gpurun_out
T="tests/test_gpu_ring.py::test_parity_build_equals_oracle_telescoped tests/test_gpu_ring.py::test_multi_packet_parity_build_equals_oracle tests/test_gpu_ring.py::test_production_against_oracle_and_literal_ring tests/test_gpu_ring.py::test_full_fill_one_packet_parity_build_equals_oracle"
K="mixed16-False or mixed8-True or mixed8-3 or mixed16] or (production and sedov16_4)"
for tool in memcheck racecheck synccheck; do
  timeout 1700 compute-sanitizer --tool $tool --kernel-regex kns=orcha --print-limit 20 \
    python -m pytest -x -q -p no:cacheprovider $T -k "$K" > gpurun_out/sanitize_ring_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/sanitize_ring_$tool.txt | tail -4
done

# compute-sanitizer over this library's kernels (fused stage kernels of both
# methods and both schemes, fill / pack / dt / device-dt kernels, the z-face
# carry, the unit kernels and the overlapped step; not the peer-mode
# barrier, whose spinning ranks need concurrent kernels the tools serialise) on
# small grids: memcheck, racecheck (shared memory hazards), synccheck
# (barrier misuse).  Summaries -> gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
T="tests/test_gpu_fillmode.py::test_gather_mode_equals_full_mode tests/test_gpu_devdt.py::test_device_dt_loop_with_scheme_variants tests/test_gpu_devdt.py::test_cuda_graph_of_device_dt_steps_equals_plain_loop tests/test_gpu_supersonic.py::test_parity_build_bitwise tests/test_gpu_unit_fuzz.py::test_riemann_flux_fuzz tests/test_gpu_multirank.py::test_overlap_step_bitwise_equal_single_domain"
K="nb1 or nb2 or scheme or graph or shear_16-0 or shear_8-1 or floor_16-0 or kw0-True or kw1-True or case0 or case2"
for tool in memcheck racecheck synccheck; do
  timeout 1700 compute-sanitizer --tool $tool --kernel-regex kns=orcha --print-limit 20 \
    python -m pytest -x -q -p no:cacheprovider $T -k "$K" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.txt | tail -4
done

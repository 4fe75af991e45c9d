# compute-sanitizer over the product path (run on a GPU box from the repo root):
#   memcheck (out-of-bounds / misaligned / leaks), initcheck (reads of
#   uninitialised device memory), racecheck and synccheck (shared memory and
#   barriers), each on smoke() and on a short GPU-test selection that covers
#   the single-GPU frame (eager, captured, replayed), the host stepFrame with
#   its overlapped download, the slab path (loopback ranks, interior/boundary
#   iteration sets), the heavy-cell sort and the component entry points.
# Summaries (ERROR SUMMARY lines) go to gpurun_out/sanitize_summary.txt.
mkdir -p gpurun_out
SEL=(tests/test_gpu_solver_behaviour.py::test_failed_frame_leaves_caller_arrays_untouched
     "tests/test_gpu_solver_behaviour.py::test_state_set_rotation_and_graph_cache_bitwise[2]"
     "tests/test_gpu_slabs.py::test_slabs_bitwise_dam_break_apbf[2]"
     tests/test_gpu_components.py::test_grid_build_bitwise
     tests/test_gpu_variants.py::test_dense_cluster_switches_to_allocated_list_slabs)
: > gpurun_out/sanitize_summary.txt
for tool in memcheck initcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
      > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "$tool smoke: $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_smoke.log | tail -1) rc=$?" >> gpurun_out/sanitize_summary.txt
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x "${SEL[@]}" \
      > gpurun_out/sanitize_${tool}_tests.log 2>&1
  echo "$tool tests: $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_tests.log | tail -1); $(grep -h 'passed\|failed' gpurun_out/sanitize_${tool}_tests.log | tail -1)" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt

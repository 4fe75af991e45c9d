# The GPU test suite on the checked build (libapbf_gpu_checked.so: -DAPBF_CHECKED
# device asserts on every data-derived index, see apbf_device.cuh).  This pool
# does not allow compute-sanitizer; a failed assert traps the kernel, which
# surfaces as a CUDA error in the test.  Run from the repo root on a GPU box.
mkdir -p gpurun_out
APBF_LIB=libapbf_gpu_checked.so python -m pytest tests -m gpu -q -p no:cacheprovider \
    --deselect tests/test_gpu_acceptance.py::test_criterion_3_wall_clock_reduction_at_1m \
    > gpurun_out/checked_tests.log 2>&1
echo "checked build rc=$?" >> gpurun_out/checked_tests.log
grep -c "APBF_DCHECK failed" gpurun_out/checked_tests.log | sed 's/^/APBF_DCHECK failures: /' >> gpurun_out/checked_tests.log
tail -4 gpurun_out/checked_tests.log

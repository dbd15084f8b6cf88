#!/bin/bash
# compute-sanitizer passes over the device path (run under gpurun).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/sanitize
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
rm -f gpurun_out/sanitize/rc.txt
if [ "${1:-all}" = "all" ]; then
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_host_e2e.py -q -x -p no:cacheprovider \
  > gpurun_out/sanitize/memcheck_pytest.txt 2>&1; echo "memcheck pytest rc=$?" >> gpurun_out/sanitize/rc.txt
for exe in tests/cpp/bin/test_mixed_gpu tests/cpp/bin/test_hmlstm_gpu tests/cpp/bin/test_user_kernel_gpu; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 $exe > gpurun_out/sanitize/memcheck_$(basename $exe).txt 2>&1; echo "memcheck $exe rc=$?" >> gpurun_out/sanitize/rc.txt
done
fi
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 tests/cpp/bin/ref_suites_b200 \
  "-tce=kernels leaking*,fused cell update matches*,all-UPDATE boundary*,reference diagonal path*,broadcast_apply reproduces the two-output*,parallel strided path matches*" \
  > gpurun_out/sanitize/memcheck_ref_suites_b200.txt 2>&1; echo "memcheck ref_suites_b200 rc=$?" >> gpurun_out/sanitize/rc.txt
for mode in k1c2 k2c2 k2c3 k2mix k2tick k2c2:r k2mix:r k2c3:r; do
  for t in racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 scripts/lab/bin/lab $mode > gpurun_out/sanitize/${t}_${mode/:/_}.txt 2>&1
    echo "$t $mode rc=$? $(grep -E 'SUMMARY' gpurun_out/sanitize/${t}_${mode/:/_}.txt | tr -s ' ')" >> gpurun_out/sanitize/rc.txt
  done
done

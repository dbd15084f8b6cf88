#!/bin/bash
# Quick GPU check of selected tests: gpu_quick.sh TAG "pytest args"
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-q}
shift
timeout 1500 python -m pytest -q -rf -x "$@" > gpurun_out/pytest_$TAG.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.txt
timeout 600 tests/cpp/bin/ref_suites_b200 > gpurun_out/ref_suites_$TAG.txt 2>&1
echo "ref_suites rc=$?" >> gpurun_out/ref_suites_$TAG.txt
timeout 300 tests/cpp/bin/test_user_kernel_gpu > gpurun_out/user_kernel_$TAG.txt 2>&1
echo "user_kernel rc=$?" >> gpurun_out/user_kernel_$TAG.txt

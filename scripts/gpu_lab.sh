#!/bin/bash
# gpu_lab.sh MODE TAG : scripts/lab/bin/lab MODE -> gpurun_out/lab_TAG.jsonl (binary built here)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout ${LAB_TIMEOUT:-900} scripts/lab/bin/lab "$1" > gpurun_out/lab_$2.jsonl 2> gpurun_out/lab_$2.err
echo "lab rc=$?" >> gpurun_out/lab_$2.err

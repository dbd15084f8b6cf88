#!/bin/bash
# Build (if needed) and run the dev tuning harness; output in gpurun_out/lab_<tag>.jsonl
cd "$(dirname "$0")/../.." || exit 1
mkdir -p scripts/lab/bin gpurun_out
if [ ! -x scripts/lab/bin/lab ] || [ scripts/lab/lab.cu -nt scripts/lab/bin/lab ]; then
  nvcc -std=c++20 -O3 --fmad=false -lineinfo -Iinclude -Ipaper_1810_08297_b200/csrc \
    -gencode arch=compute_100a,code=sm_100a scripts/lab/lab.cu -o scripts/lab/bin/lab || exit 1
fi
timeout ${LAB_TIMEOUT:-600} scripts/lab/bin/lab "${1:-all}" > gpurun_out/lab_${2:-run}.jsonl 2> gpurun_out/lab_${2:-run}.err
echo "lab rc=$?"

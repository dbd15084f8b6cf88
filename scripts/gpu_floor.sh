#!/bin/bash
# Config-2 memory-floor probes (scripts/lab/floor.cu) + K1 itself at the same size (lab "floor").
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 scripts/lab/bin/floor > gpurun_out/lab_floor_bulk.jsonl 2> gpurun_out/lab_floor_bulk.err
echo "floor rc=$?"
LAB_TIMEOUT=300 bash scripts/lab/run.sh floor floor_k1

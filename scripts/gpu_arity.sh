#!/bin/bash
# K1 arity variants (lab_ar0/1/2 = pipeline, no pipeline, no pipeline + >= 3 CTAs/SM for A >= 16)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 0 1 2; do timeout 600 scripts/lab/bin/lab_ar$v arity > gpurun_out/lab_arity_v$v.jsonl 2>&1; done

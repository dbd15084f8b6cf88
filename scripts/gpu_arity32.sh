#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 0 2; do timeout 600 scripts/lab/bin/lab_ar$v arity32 > gpurun_out/lab_arity32_v$v.jsonl 2>&1; done

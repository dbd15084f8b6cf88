cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do
timeout 600 scripts/lab/bin/lab k2r5 >> gpurun_out/lab_k2r5_skip.jsonl 2>&1
timeout 600 scripts/lab/bin/lab_noskip k2r5 >> gpurun_out/lab_k2r5_noskip.jsonl 2>&1
done

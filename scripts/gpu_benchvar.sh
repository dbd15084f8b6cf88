cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for K in 30 30 60 120; do timeout 300 python bench.py --steps $K --warmup 5 --extra none --no-cpu-baseline --e2e-steps 2 >> gpurun_out/bench_var.jsonl 2>> gpurun_out/bench_var.err; done

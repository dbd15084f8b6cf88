cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python scripts/reduced_probe.py > gpurun_out/reduced_probe.jsonl 2> gpurun_out/reduced_probe.err
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -rf > gpurun_out/multirank.txt 2>&1

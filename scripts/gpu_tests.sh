#!/bin/bash
# Full GPU test pass + smoke (used by the round's gpurun calls).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
for exe in tests/cpp/bin/test_*; do timeout 300 "$exe" > "gpurun_out/$(basename $exe).txt" 2>&1; done

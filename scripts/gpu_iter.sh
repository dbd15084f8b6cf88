#!/bin/bash
# One build->measure iteration under gpurun: GPU tests, C++ tests, smoke, bench, launch list, ncu full (cfg2).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-iter}
nvidia-smi > gpurun_out/nvidia_smi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40 > gpurun_out/pytest_gpu_$TAG.txt
for exe in tests/cpp/bin/test_*; do timeout 300 "$exe" > "gpurun_out/$(basename $exe)_$TAG.txt" 2>&1; echo "$exe rc=$?" >> gpurun_out/cpp_rc_$TAG.txt; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
if [ "${2:-}" != "noprof" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fwd2d|pull2d" -c 12 --csv --log-file gpurun_out/launches_cfg2_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra "" --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d" -s 4 -c 2 -o gpurun_out/prof_cfg2_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra "" --e2e-steps 1 > /dev/null 2>&1
fi
ls gpurun_out

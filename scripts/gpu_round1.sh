#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fwd2d|pull2d" -c 12 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra "" --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d" -s 4 -c 2 -o gpurun_out/prof_cfg2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra "" --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d" -s 4 -c 2 -o gpurun_out/prof_cfg5 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --extra "" --e2e-steps 1 > gpurun_out/ncu_full5.log 2>&1
ls -la gpurun_out

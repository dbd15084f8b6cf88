#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; one GPU, single-process commands only).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/prof
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra none --e2e-steps 1 --graph 0"
# 1. launch list of the bench command (every kernel, cold-cache serialised)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches_cfg2.csv $B --config cfg2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fwd2d|pull2d|pull_finish" --csv --log-file gpurun_out/prof/launches_cfg5.csv $B --config cfg5 > /dev/null 2>&1
# 2. full captures of K1 and K2
for c in cfg2 cfg3 cfg5 cfg4div; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d|pull_finish" -s 6 -c 2 -f -o gpurun_out/prof/full_$c $B --config $c > /dev/null 2>&1
done
ls -la gpurun_out/prof

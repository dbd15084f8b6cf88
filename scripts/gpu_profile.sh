#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; one GPU, single-process commands only).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/prof
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra none --e2e-steps 1 --graph 0"
# 1. launch list of the bench command (every kernel, cold-cache serialised)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches_cfg2.csv $B --config cfg2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fwd2d|pull2d|pull_finish" --csv --log-file gpurun_out/prof/launches_cfg5.csv $B --config cfg5 > /dev/null 2>&1
# 2. full captures of K1 and K2 (K2f too); raw / details / SASS-source pages exported
#    here as gzipped CSV, reports dropped (gpurun's 64 MiB merge limit)
for c in cfg2 cfg3 cfg5 cfg4div; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d|pull_finish" -s 6 -c 3 -f -o gpurun_out/prof/full_$c $B --config $c > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d|pull_finish" -s 2 -c 3 -f -o gpurun_out/prof/full_cfg5r python scripts/k2r_probe.py > /dev/null 2>&1
for A in 16 32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd2d -s 2 -c 1 -f -o gpurun_out/prof/full_arity$A python scripts/arity_probe.py $A > /dev/null 2>&1
done
for r in gpurun_out/prof/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i "$r" --page raw --csv 2>/dev/null | gzip > $b.raw.csv.gz
  ncu -i "$r" --page details --csv 2>/dev/null | gzip > $b.details.csv.gz
  ncu -i "$r" --page source --csv --print-source sass 2>/dev/null | gzip > $b.source.csv.gz
  rm -f "$r"
done
ls -la gpurun_out/prof

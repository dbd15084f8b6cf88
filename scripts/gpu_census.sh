#!/bin/bash
# Transcendental census: ncu source-level SASS counts of K1 per boundary case.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/census; mkdir -p $O
for form in canonical select; do
  for case in copy update flush random; do
    timeout 300 ncu --set full --import-source on --clock-control none -k regex:fwd2d -c 1 -f -o $O/k1_${form}_${case} python scripts/census.py $form $case > /dev/null 2>&1
    ncu -i $O/k1_${form}_${case}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/k1_${form}_${case}.sass.csv.gz
    ncu -i $O/k1_${form}_${case}.ncu-rep --page raw --csv --metrics smsp__inst_executed.sum,smsp__inst_executed_pipe_xu.sum,sm__sass_thread_inst_executed_op_mufu? 2>/dev/null | gzip > $O/k1_${form}_${case}.raw.csv.gz
    rm -f $O/k1_${form}_${case}.ncu-rep
  done
done
ls -la $O

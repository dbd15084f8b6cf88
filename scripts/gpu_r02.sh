#!/bin/bash
# Round-2 iteration: GPU tests, smoke, bench (+ reference arm), optional ncu captures.
# gpu_r02.sh TAG [ncu-target...]   ncu targets: arity | cfg2 | cfg3 | census
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/$1
O=gpurun_out/$1
nvidia-smi > $O/nvidia_smi.txt 2>&1
[ "${SKIP_BASE:-0}" = 1 ] || {
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
}
shift
for t in "$@"; do
  case $t in
    arity) timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd2d -c 2 -s 2 -o $O/ncu_arity16 -f python scripts/arity_probe.py 16 > /dev/null 2>&1
           timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd2d -c 2 -s 2 -o $O/ncu_arity32 -f python scripts/arity_probe.py 32 > /dev/null 2>&1 ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra none --e2e-steps 1 --graph 0 > /dev/null 2>&1 ;;
    cfg3) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d|pull_finish" -s 6 -c 3 -f -o $O/ncu_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra none --e2e-steps 1 --graph 0 --config cfg3 > /dev/null 2>&1 ;;
    cfg5r) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pull2d" -s 1 -c 1 -f -o $O/ncu_cfg5r python scripts/k2r_probe.py > $O/ncu_cfg5r.log 2>&1 ;;
    cfg2) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd2d|pull2d" -s 6 -c 2 -f -o $O/ncu_cfg2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra none --e2e-steps 1 --graph 0 --config cfg2 > /dev/null 2>&1 ;;
  esac
done
# keep the merge under gpurun's 64 MiB: raw/details pages as gzipped CSV, reports only when small
for r in $O/*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i "$r" --page raw --csv 2>/dev/null | gzip > $b.raw.csv.gz
  ncu -i "$r" --page details --csv 2>/dev/null | gzip > $b.details.csv.gz
  ncu -i "$r" --page source --csv --print-source sass 2>/dev/null | gzip > $b.source.csv.gz
  [ $(stat -c %s "$r") -gt 12000000 ] && rm -f "$r"
done
du -sh $O; ls -la $O

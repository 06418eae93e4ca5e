#!/bin/bash
# Final-session GPU pass: suite, smoke, bench, reference arm, then (each after its
# command exited 0 without ncu) one ncu --set full capture of the headline fold
# (1024-thread CTAs) and the bench command's launch list.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
(python -m pytest tests -m gpu -q 2>&1 | tail -30) > gpurun_out/gpu_tests.log
echo "pytest rc=${PIPESTATUS[0]}" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
P="python tools/profile_case.py"
$P --steps 1 > gpurun_out/p1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fold_once -c 1 \
      -o gpurun_out/r2c_fold_once -f $P --steps 1 > gpurun_out/n1.log 2>&1
echo "fold ncu rc=$?"
ncu -i gpurun_out/r2c_fold_once.ncu-rep --page raw --csv > gpurun_out/r2c_fold_once_raw.csv 2>/dev/null
ncu -i gpurun_out/r2c_fold_once.ncu-rep --page details --csv > gpurun_out/r2c_fold_once_details.csv 2>/dev/null
rm -f gpurun_out/r2c_fold_once.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches_bench.csv \
    python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ncu.json 2> gpurun_out/bench_ncu.err
echo "launch list rc=$?"
tail -2 gpurun_out/gpu_tests.log

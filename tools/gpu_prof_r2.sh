#!/bin/bash
# round-2 ncu evidence (one gpurun call = one ncu "use"): each profiled command
# first exits 0 without ncu, then runs under ncu; the reports are exported to
# CSV on the box and deleted (gpurun copies back at most 64 MiB).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
P="python tools/profile_case.py"
N="ncu --set full --clock-control none --import-source on"
exp() {  # export a report's raw metrics + details, then drop the .ncu-rep
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
$P --steps 1 > gpurun_out/p1.log 2>&1 && \
  $N -k regex:fold_once -c 1 -o gpurun_out/r2_fold_once -f $P --steps 1 > gpurun_out/n1.log 2>&1
echo "fold rc=$?"; exp r2_fold_once
$P --loopback --steps 2 > gpurun_out/p2.log 2>&1 && \
  $N -k regex:loopback_allreduce -s 1 -c 1 -o gpurun_out/r2_loopback_allreduce -f $P --loopback --steps 2 > gpurun_out/n2.log 2>&1
echo "loopback rc=$?"; exp r2_loopback_allreduce
$P --op allgather --ragged --steps 1 > gpurun_out/p3.log 2>&1 && \
  $N -k regex:fanout_shift -c 1 -o gpurun_out/r2_fanout_shift -f $P --op allgather --ragged --steps 1 > gpurun_out/n3.log 2>&1
echo "fanout_shift rc=$?"; exp r2_fanout_shift
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err
echo "bench plain rc=$?"; tail -c 1500 gpurun_out/bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ncu.json 2> gpurun_out/bench_ncu.err
echo "launch list rc=$?"; tail -c 1500 gpurun_out/bench_ncu.err
du -sh gpurun_out

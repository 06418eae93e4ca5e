#!/bin/bash
# ncu (full set) of the loopback rank kernels with the bulk-copy copy phases:
# AllReduce fp32 8 x 256 MiB and AllGather bf16 (256 MiB gathered).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
P="python tools/profile_case.py"
N="ncu --set full --clock-control none --import-source on"
exp() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/$1_raw.csv > gpurun_out/$1_summary.txt
  rm -f gpurun_out/$1.ncu-rep
}
$P --loopback --steps 2 > gpurun_out/pb1.log 2>&1 && \
  $N -k regex:loopback_allreduce -s 1 -c 1 -o gpurun_out/r2_loopback_allreduce_bulk -f $P --loopback --steps 2 > gpurun_out/nb1.log 2>&1
echo "allreduce rc=$?"; exp r2_loopback_allreduce_bulk
$P --loopback --op allgather --steps 2 > gpurun_out/pb2.log 2>&1 && \
  $N -k regex:loopback_allgather -s 1 -c 1 -o gpurun_out/r2_loopback_allgather_bulk -f $P --loopback --op allgather --steps 2 > gpurun_out/nb2.log 2>&1
echo "allgather rc=$?"; exp r2_loopback_allgather_bulk
cat gpurun_out/r2_loopback_allreduce_bulk_summary.txt gpurun_out/r2_loopback_allgather_bulk_summary.txt

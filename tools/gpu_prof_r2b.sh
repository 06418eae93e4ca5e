#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
P="python tools/profile_case.py"
N="ncu --set full --clock-control none --import-source on"
exp() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
$P --loopback --steps 2 > gpurun_out/p2.log 2>&1 && \
  $N -k regex:loopback_allreduce -s 1 -c 1 -o gpurun_out/r2_loopback_allreduce_staggered -f $P --loopback --steps 2 > gpurun_out/n2.log 2>&1
echo "loopback rc=$?"; exp r2_loopback_allreduce_staggered
$P --loopback --op reducescatter --steps 2 > gpurun_out/p3.log 2>&1 && \
  $N -k regex:loopback_reducescatter -s 1 -c 1 -o gpurun_out/r2_loopback_reducescatter -f $P --loopback --op reducescatter --steps 2 > gpurun_out/n3.log 2>&1
echo "rs rc=$?"; exp r2_loopback_reducescatter

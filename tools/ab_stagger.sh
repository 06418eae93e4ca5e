#!/bin/bash
# A/B of the staggered-round schedule on the loopback engine: the shipped
# library vs a variant built with the round-1 schedule (one round, in step).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python tools/loopback_bench.py 8,4 all > gpurun_out/ab_new.jsonl 2>&1
python tools/build_variant.py /tmp/flx_r1sched -DFLX_ROUNDS_PER_CALL=1 -DFLX_STAGGER=0 > gpurun_out/ab_build.log 2>&1 || { tail -n 20 gpurun_out/ab_build.log; exit 1; }
FLEXLINK_LIBRARY=/tmp/flx_r1sched/libflexlink.so python tools/loopback_bench.py 8,4 all > gpurun_out/ab_old.jsonl 2>&1
python -m pytest tests/test_gpu_loopback.py tests/test_gpu_sequence.py tests/test_gpu_fuzz.py tests/test_gpu_reducescatter.py tests/test_gpu_ipc_loopback.py -x -q > gpurun_out/pt.log 2>&1; echo "tests rc=$?"
tail -n 2 gpurun_out/pt.log
echo new; cat gpurun_out/ab_new.jsonl; echo old; cat gpurun_out/ab_old.jsonl

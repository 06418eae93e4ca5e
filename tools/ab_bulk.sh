#!/bin/bash
# A/B of the rank kernels' copy phases on the loopback engine: TMA bulk copies
# through a dynamic shared-memory ring (default) vs register copies
# (FLX_BULK=0), alternating, twice; optional variants built with
# tools/build_variant.py -DFLX_BULK_TILE=.. -DFLX_BULK_STAGES=.. into build/var_*;
# then the whole GPU suite on the default.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: > gpurun_out/ab_bulk.jsonl
for rep in 1 2; do
  for mode in 1 0; do
    FLX_BULK=$mode python tools/loopback_bench.py 8,4,2 | sed "s/^{/{\"bulk\": $mode, \"rep\": $rep, /" >> gpurun_out/ab_bulk.jsonl
    FLX_BULK=$mode python tools/loopback_bench.py 8,4 all | sed "s/^{/{\"bulk\": $mode, \"rep\": $rep, /" >> gpurun_out/ab_bulk.jsonl
  done
  for v in build/var_*/; do
    [ -e "$v/libflexlink.so" ] || continue
    name=$(basename "$v")
    FLEXLINK_LIBRARY=$v/libflexlink.so python tools/loopback_bench.py 8,4,2 | sed "s/^{/{\"bulk\": \"$name\", \"rep\": $rep, /" >> gpurun_out/ab_bulk.jsonl
    FLEXLINK_LIBRARY=$v/libflexlink.so python tools/loopback_bench.py 8,4 all | sed "s/^{/{\"bulk\": \"$name\", \"rep\": $rep, /" >> gpurun_out/ab_bulk.jsonl
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_bulk_default.log 2>&1
echo "suite rc=$? $(tail -n 1 gpurun_out/pt_bulk_default.log)"
FLX_BULK=0 timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_fuzz.py tests/test_gpu_sequence.py tests/test_gpu_reducescatter.py -x -q > gpurun_out/pt_bulk_off.log 2>&1
echo "bulk-off parity rc=$? $(tail -n 1 gpurun_out/pt_bulk_off.log)"

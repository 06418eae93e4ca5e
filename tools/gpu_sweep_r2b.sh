#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python tools/sweep_c3.py --inlib --nvlink-ctas 3 --steps 20 --warmup 5 --max-mib 64 > gpurun_out/c3b_capped.jsonl 2> gpurun_out/c3b_capped.err; echo "capped rc=$?"
python tools/sweep_c3.py --inlib --loopback --nvlink-ctas 1 --max-mib 64 --ranks 2,4 --steps 10 --warmup 3 > gpurun_out/c3b_lb.jsonl 2> gpurun_out/c3b_lb.err; echo "loopback rc=$?"
python -m pytest tests/test_gpu_autotune.py -q > gpurun_out/at.log 2>&1; echo "autotune tests rc=$?"

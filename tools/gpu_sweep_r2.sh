#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python tools/sweep_c3.py --inlib --nvlink-ctas 3 --steps 20 --warmup 5 > gpurun_out/c3_inlib_capped.jsonl 2> gpurun_out/c3_capped.err; echo "capped rc=$?"
python tools/sweep_c3.py --inlib --steps 20 --warmup 5 > gpurun_out/c3_inlib_uncapped.jsonl 2> gpurun_out/c3_uncapped.err; echo "uncapped rc=$?"
python tools/sweep_c3.py --inlib --loopback --nvlink-ctas 1 --max-mib 256 --ranks 2,4,8 --steps 10 --warmup 3 > gpurun_out/c3_inlib_loopback_capped.jsonl 2> gpurun_out/c3_lb.err; echo "loopback rc=$?"
tail -3 gpurun_out/c3_capped.err gpurun_out/c3_uncapped.err gpurun_out/c3_lb.err
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err
echo "bench plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ncu.json 2> gpurun_out/bench_ncu.err
echo "launch list rc=$?"; tail -c 800 gpurun_out/bench_ncu.err

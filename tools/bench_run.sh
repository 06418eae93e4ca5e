#!/bin/bash
# gpurun helper: one bench line (+ optional pytest selection)
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
if [ -n "$PYTEST_SEL" ]; then
  python -m pytest $PYTEST_SEL -x -q > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
  tail -3 gpurun_out/pytest_sel.log
fi
python bench.py --steps ${STEPS:-20} --warmup ${WARMUP:-5} $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"; cat gpurun_out/bench_ref.json | head -c 400

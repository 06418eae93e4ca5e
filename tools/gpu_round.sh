#!/bin/bash
# One gpurun call: GPU test suite, smoke, smoke launch list.  Usage:
#   gpurun --timeout 1800 -- bash tools/gpu_round.sh [pytest-args]
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -5 gpurun_out/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log

#!/bin/bash
# round-2 GPU check: full GPU suite, NVLS diagnosis, loopback occupancy, bench
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python tools/nvls_diag.py > gpurun_out/nvls_diag.json 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2510_15882_b200 import comm; print(comm.nvls_probe(0))" > gpurun_out/nvls_probe.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -3 gpurun_out/pytest.log
python tools/loopback_bench.py 8,4,2 > gpurun_out/lb.jsonl 2> gpurun_out/lb.err
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"

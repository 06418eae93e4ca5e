#!/bin/bash
# The bench command's own run, then the ncu launch list of the same command
# (gpu__time_duration.sum per launch, --clock-control none), summarised.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ll.json 2> gpurun_out/bench_ll.err
echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ncu.out 2> gpurun_out/bench_ncu.err
echo "launch list rc=$?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/launches_bench.csv")) if len(r) > 14 and r[0].isdigit()]
t = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    t[r[4]][0] += 1
    t[r[4]][1] += float(r[14].replace(",", ""))
tot = sum(v[1] for v in t.values())
print("launches", len(rows), "total_ms", round(tot / 1e6, 2))
for k, (n, ns) in sorted(t.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{n:6d} {ns / 1e6:10.2f} ms {100 * ns / tot:5.1f}%  {k[:110]}")
PY

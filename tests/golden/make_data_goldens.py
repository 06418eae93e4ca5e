"""Generate tests/golden/data_plane.json: order-independent data fixtures.

The reference moves no bytes, so its data plane has no golden vectors
(SURVEY.md §8c).  These fixtures pin what any correct striped collective must
produce regardless of reduction order or path split:

* AllReduce sum over small integer-valued fp32/bf16/int32 inputs — the exact
  mathematical sum, computed here with Python integers;
* AllReduce max/min over arbitrary values — order-independent by definition;
* AllGather — plain concatenation;
* the per-path byte split of each case, taken from the REFERENCE's own
  ``linkstripe.partition`` (imported from /root/reference/pkg/src).

Run in the build container:  python tests/golden/make_data_goldens.py
"""

import json
import random
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "data_plane.json"


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import linkstripe as ls

    rng = random.Random(7)
    cases = []
    specs = [  # (op, dtype, esz, nranks, count, granules, alignment)
        ("allreduce_sum", 7, 4, 8, 2048, (854, 146, 0), 4096),
        ("allreduce_sum", 7, 4, 3, 1001, (1000, 0, 0), 3 * 4096),
        ("allreduce_sum", 9, 2, 8, 4096, (500, 500, 0), 4096),
        ("allreduce_sum", 2, 4, 5, 777, (600, 400, 0), 16),
        ("allreduce_max", 7, 4, 4, 2048, (750, 250, 0), 4096),
        ("allreduce_min", 2, 4, 6, 999, (1000, 0, 0), 1),
        ("allgather", 1, 1, 4, 9001, (500, 500, 0), 4096),
        ("allgather", 9, 2, 8, 1500, (1000, 0, 0), 4096),
    ]
    for op, dtype, esz, n, count, g, align in specs:
        if dtype == 9:  # bf16 holds integers up to 256 exactly; keep |sum| <= 256
            ranks = [[rng.randint(-32, 32) for _ in range(count)] for _ in range(n)]
        elif op == "allreduce_max" or op == "allreduce_min":
            ranks = [[rng.randint(-10**6, 10**6) for _ in range(count)] for _ in range(n)]
        elif dtype == 1:
            ranks = [[rng.randint(0, 255) for _ in range(count)] for _ in range(n)]
        else:
            ranks = [[rng.randint(-4096, 4096) for _ in range(count)] for _ in range(n)]
        if op == "allreduce_sum":
            expect = [sum(col) for col in zip(*ranks)]
        elif op == "allreduce_max":
            expect = [max(col) for col in zip(*ranks)]
        elif op == "allreduce_min":
            expect = [min(col) for col in zip(*ranks)]
        else:
            expect = [x for r in ranks for x in r]
        size = count * esz
        split = ls.partition(size, {ls.PathKind(i): v for i, v in enumerate(g)}, align)
        cases.append({"op": op, "dtype": dtype, "nranks": n, "count": count,
                      "granules": list(g), "alignment": align, "inputs": ranks,
                      "expect": expect,
                      "split": [split.get(ls.PathKind(i), 0) for i in range(3)]})
    OUT.write_text(json.dumps({"source": "exact arithmetic + linkstripe.partition",
                               "cases": cases}))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()

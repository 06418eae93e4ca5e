"""The CPU data oracle, pinned before it is trusted (no GPU needed).

* against tests/golden/data_plane.json (exact sums / max / min / concatenation
  and the reference's own partition split);
* against an independent numpy statement of the fold rule;
* its bf16/fp16 rounding against torch / numpy conversions.
"""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle

DATA = json.loads((Path(__file__).parent / "golden" / "data_plane.json").read_text())
NP = {1: np.uint8, 2: np.int32, 7: np.float32}


def _encode(values, dtype):
    if dtype == 9:
        return oracle.f32_to_bf16_bits(np.asarray(values, dtype=np.float32))
    return np.asarray(values, dtype=NP[dtype])


def _decode(arr, dtype):
    if dtype == 9:
        return oracle.bf16_bits_to_f32(arr).astype(np.int64)
    return arr.astype(np.int64)


@pytest.mark.parametrize("case", DATA["cases"], ids=lambda c: f"{c['op']}-{c['dtype']}")
def test_oracle_reproduces_golden_data(case):
    n, dtype = case["nranks"], case["dtype"]
    assert oracle.partition(case["count"] * (2 if dtype == 9 else np.dtype(NP.get(dtype, np.uint8)).itemsize),
                            case["granules"], case["alignment"]) == case["split"]
    sends = [_encode(r, dtype) for r in case["inputs"]]
    if case["op"] == "allgather":
        out = oracle.allgather(sends, dtype, case["granules"], case["alignment"])
    else:
        op = {"allreduce_sum": oracle.SUM, "allreduce_max": oracle.MAX,
              "allreduce_min": oracle.MIN}[case["op"]]
        out = oracle.allreduce(sends, dtype, op, case["granules"], case["alignment"])
    for r in range(n):
        np.testing.assert_array_equal(_decode(out[r], dtype), np.asarray(case["expect"]))


def _rand(dtype, n, count, rng):
    if dtype == 9 or dtype == 6:
        x = (rng.standard_normal(count * n) * 3).astype(np.float32)
        bits = oracle.f32_to_bf16_bits(x) if dtype == 9 else x.astype(np.float16).view(np.uint16)
        return [bits[i * count:(i + 1) * count].copy() for i in range(n)]
    if dtype in (7, 8):
        t = np.float32 if dtype == 7 else np.float64
        return [(rng.standard_normal(count) * 3).astype(t) for _ in range(n)]
    t = oracle.DTYPES[dtype]
    info = np.iinfo(t)
    return [rng.integers(info.min, info.max, count, dtype=t, endpoint=True) for _ in range(n)]


@pytest.mark.parametrize("dtype", list(range(10)))
@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_c_oracle_matches_numpy_fold(dtype, op):
    rng = np.random.default_rng(dtype * 10 + op)
    sends = _rand(dtype, 5, 3001, rng)
    want = oracle.fold_numpy(sends, dtype, op)
    got = oracle.allreduce(sends, dtype, op, (700, 300, 0), 1 * 16)
    for r in got:
        if dtype in (6, 7, 8, 9):
            np.testing.assert_array_equal(r.view(np.uint8), np.asarray(want).view(np.uint8))
        else:
            np.testing.assert_array_equal(r, want)


def test_oracle_in_place_and_shares_do_not_change_bits():
    rng = np.random.default_rng(3)
    sends = _rand(7, 8, 50000, rng)
    ref = oracle.allreduce(sends, 7, oracle.SUM, (1000, 0, 0), 1)
    for g in ((854, 146, 0), (500, 300, 200), (1, 999, 0)):
        got = oracle.allreduce(sends, 7, oracle.SUM, g, 8 * 16)
        np.testing.assert_array_equal(got[0], ref[0])
    inplace = [s.copy() for s in sends]
    oracle.allreduce(inplace, 7, oracle.SUM, (900, 100, 0), 8 * 16, recvs=inplace)
    for r in inplace:
        np.testing.assert_array_equal(r, ref[0])


def test_bf16_and_fp16_rounding_match_torch_and_numpy():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.standard_normal(200000).astype(np.float32) * 1e3,
                        rng.standard_normal(1000).astype(np.float32) * 1e-6,
                        np.array([0.0, -0.0, 65504.0, 65519.0, 65520.0, 1e-8, 6e-8, 3e38],
                                 dtype=np.float32)])
    L = oracle.lib()
    want_bf = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got_bf = np.array([L.flxo_f32_to_bf16(float(v)) for v in x[:5000]], dtype=np.uint16)
    np.testing.assert_array_equal(got_bf, want_bf[:5000])
    np.testing.assert_array_equal(oracle.f32_to_bf16_bits(x), want_bf)
    small = x[np.abs(x) < 70000]
    want_h = small.astype(np.float16).view(np.uint16)
    got_h = np.array([L.flxo_f32_to_f16(float(v)) for v in small[:20000]], dtype=np.uint16)
    np.testing.assert_array_equal(got_h, want_h[:20000])
    tail = small[-8:]
    np.testing.assert_array_equal(np.array([L.flxo_f32_to_f16(float(v)) for v in tail],
                                           dtype=np.uint16), tail.astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("dtype", [0, 2, 6, 7, 8, 9])
@pytest.mark.parametrize("op", [0, 2])
def test_reducescatter_oracle_matches_numpy(dtype, op):
    rng = np.random.default_rng(100 + dtype + op)
    n, count = 5, 1237
    sends = _rand(dtype, n, n * count, rng)
    got = oracle.reducescatter(sends, dtype, op, (600, 400, 0), 16)
    for r in range(n):
        want = oracle.fold_numpy([s[r * count:(r + 1) * count] for s in sends], dtype, op)
        np.testing.assert_array_equal(np.asarray(got[r]).view(np.uint8),
                                      np.asarray(want).view(np.uint8))
    # reduce_scatter == the matching block of an all_reduce
    full = oracle.allreduce(sends, dtype, op)
    for r in range(n):
        np.testing.assert_array_equal(np.asarray(got[r]).view(np.uint8),
                                      full[0][r * count:(r + 1) * count].view(np.uint8))


def test_alltoall_oracle_is_a_block_transpose():
    rng = np.random.default_rng(5)
    n, count = 4, 999
    sends = [rng.integers(0, 255, n * count, dtype=np.uint8) for _ in range(n)]
    got = oracle.alltoall(sends, 1, (700, 300, 0), 16)
    for q in range(n):
        want = np.concatenate([sends[r][q * count:(q + 1) * count] for r in range(n)])
        np.testing.assert_array_equal(got[q], want)


def test_oracle_rejects_bad_arguments():
    with pytest.raises(ValueError):
        oracle.partition(10, (500, 400, 0), 0)
    with pytest.raises(ValueError):
        oracle.allreduce([np.zeros(4, np.float32)], 7, 9)
    with pytest.raises(ValueError):  # slice boundary inside an element
        oracle.allreduce([np.zeros(5, np.float32)] * 2, 7, 0, (500, 500, 0), 2)

"""Where the host time of one small 8-virtual-rank call goes (Python side)."""
import ctypes
import json
import os
import sys
import timeit

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402

n = 8
cl = flx.Clique(n)
s = [torch.randn(1024, device="cuda") for _ in range(n)]
r = [torch.empty_like(x) for x in s]
L = flx.load_library()
ptrs = ctypes.c_void_p * n
stream = flx._stream_handle(None)
sp = ptrs(*[t.data_ptr() for t in s])
rp = ptrs(*[t.data_ptr() for t in r])
N = 2000


def us(fn):
    fn()
    return round(timeit.timeit(fn, number=N) / N * 1e6, 2)


out = {
    "full all_reduce": us(lambda: cl.all_reduce(s, r)),
    "validate (cached)": us(lambda: cl._validate(s, r)),
    "ptr arrays": us(lambda: (ptrs(*[t.data_ptr() for t in s]), ptrs(*[t.data_ptr() for t in r]))),
    "stream handle": us(lambda: flx._stream_handle(None)),
    "dtype_code": us(lambda: flx.dtype_code(s[0].dtype)),
    "ctypes flxGroupCollective only": us(lambda: L.flxGroupCollective(0, cl._handles, n, sp, rp,
                                                                     1024, 7, 0, stream)),
    "ctypes flxGetVersion": us(lambda: L.flxGetVersion(ctypes.byref(ctypes.c_int()))),
}
torch.cuda.synchronize()
print(json.dumps(out))

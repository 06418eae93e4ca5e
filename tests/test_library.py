"""The C-ABI library loads and exports every entry point include/flexlink.h declares.

Runs without a GPU: no collective is executed, but the no-GPU behaviour of the
product path is pinned (it fails loudly, it never falls back to the CPU).
"""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2510_15882_b200 import comm

ROOT = Path(__file__).resolve().parents[1]
HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared():
    names = set()
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"^\s*(?:const\s+)?[\w]+\**\s+\**(flx\w+|nccl\w+)\s*\(", text,
                                re.M))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2510_15882_b200.build import build

    build()
    return comm.load_library()


def test_headers_declare_the_nccl_shaped_surface():
    names = declared()
    for must in ("flxGetUniqueId", "flxCommInitRank", "flxCommInitAll", "flxCommDestroy",
                 "flxAllReduce", "flxAllGather", "flxGroupStart", "flxGroupEnd", "flxSetShares",
                 "flxGetPathTimes", "flxSetNvlinkCtas"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    path = comm.library_path()
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = sorted(declared() - exported)
    assert not missing, f"declared but not exported: {missing}"
    for name in declared():
        assert getattr(lib, name) is not None


def test_library_targets_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(comm.library_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_version_errors_and_unique_id(lib):
    v = ctypes.c_int()
    assert lib.flxGetVersion(ctypes.byref(v)) == 0 and v.value == 10000
    assert lib.flxGetErrorString(4) == b"invalid argument"
    uid = comm.Communicator.unique_id()
    assert len(uid) == 128 and uid[:4] == b"FLX1"
    assert comm.Communicator.unique_id() != uid


def test_no_gpu_means_loud_failure_not_fallback(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(comm.FlexLinkError):
        comm.Clique(2)
    handles = (ctypes.c_void_p * 1)()
    rc = lib.flxCommInitAll(handles, 1, None)
    assert rc == 1  # flxUnhandledCudaError
    assert lib.flxGetLastError()


def test_argument_validation_without_device(lib):
    assert lib.flxAllReduce(None, None, 0, 7, 0, None, None) == 4
    assert lib.flxGroupEnd() == 5  # unbalanced
    g = (ctypes.c_int * 3)(1000, 0, 0)
    assert lib.flxSetShares(None, 0, -2, g) == 4


def test_nccl_shim_exports_nccl_named_entry_points(lib):
    shim = comm.library_path().parent / "libflexlink_nccl.so"
    if not shim.exists():
        pytest.skip("/usr/include/nccl.h absent: shim not built")
    out = subprocess.run(["nm", "-D", "--defined-only", str(shim)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in ("ncclGetUniqueId", "ncclCommInitRank", "ncclCommInitAll", "ncclCommDestroy",
                 "ncclAllReduce", "ncclAllGather", "ncclReduceScatter", "ncclGroupStart",
                 "ncclGroupEnd", "ncclCommGetAsyncError", "ncclCommAbort",
                 "ncclCommFinalize", "ncclCommSplit", "ncclBroadcast", "ncclBcast",
                 "ncclAlltoAll", "ncclReduce", "ncclGather", "ncclScatter"):
        assert name in exported
    # comm-taking NCCL calls FlexLink does not implement are defined and refused,
    # so a preloaded process never hands a FlexLink comm to the real libnccl
    for name in ("ncclSend", "ncclRecv", "ncclCommShrink", "ncclCommRegister",
                 "ncclDevCommCreate", "ncclDevCommDestroy"):
        assert name in exported
    # the config-taking inits frameworks use create FlexLink communicators
    assert "ncclCommInitRankConfig" in exported and "ncclCommInitRankScalable" in exported
    # ...while comm-less calls FlexLink does not provide still resolve to NCCL
    assert "ncclMemAlloc" not in exported and "ncclGroupSimulateEnd" not in exported
    S = ctypes.CDLL(str(shim))
    S.ncclGetErrorString.restype = ctypes.c_char_p
    assert S.ncclGetErrorString(4) == b"invalid argument"
    uid = (ctypes.c_char * 128)()
    assert S.ncclGetUniqueId(uid) == 0 and bytes(uid)[:4] == b"FLX1"
    # a handle that is not a live FlexLink communicator (e.g. a real ncclComm_t)
    # is rejected by its magic word instead of being used
    fake = (ctypes.c_uint64 * 64)()
    n = ctypes.c_int()
    assert S.ncclCommCount(ctypes.byref(fake), ctypes.byref(n)) == 4
    S.ncclGetLastError.restype = ctypes.c_char_p
    assert b"not a live FlexLink communicator" in S.ncclGetLastError(None)
    assert S.ncclBroadcast(None, None, 0, 7, 0, ctypes.byref(fake), None) == 4
    assert S.ncclAllReduce(None, None, 0, 7, 0, ctypes.byref(fake), None) == 4
    # a config not set up with NCCL_CONFIG_INITIALIZER is refused before any
    # bootstrap (NCCL's rule), and so is a Scalable init without unique ids
    class UniqueId(ctypes.Structure):  # ncclUniqueId is passed by value
        _fields_ = [("internal", ctypes.c_char * 128)]

    raw = (ctypes.c_uint64 * 16)()
    out_comm = ctypes.c_void_p()
    S.ncclCommInitRankConfig.argtypes = [ctypes.c_void_p, ctypes.c_int, UniqueId, ctypes.c_int,
                                         ctypes.c_void_p]
    assert S.ncclCommInitRankConfig(ctypes.byref(out_comm), 2, UniqueId(bytes(uid)), 0,
                                    ctypes.byref(raw)) == 4
    assert b"NCCL_CONFIG_INITIALIZER" in S.ncclGetLastError(None)
    assert S.ncclCommInitRankScalable(ctypes.byref(out_comm), 2, 0, 0, None, None) == 4


def test_header_is_plain_c_and_links(tmp_path, lib):
    # the C-ABI is consumable from C (a cgo / FFI caller's view): strict C11,
    # -pedantic, no C++ in the header; link and call the no-device entry points
    src = tmp_path / "caller.c"
    src.write_text(
        '#include "flexlink.h"\n#include <stdio.h>\n#include <string.h>\n'
        "int main(void) {\n"
        "  int v = 0; flxUniqueId id; memset(&id, 0, sizeof id);\n"
        "  if (flxGetVersion(&v) != flxSuccess || v != FLX_VERSION_CODE) return 1;\n"
        "  if (flxGetUniqueId(&id) != flxSuccess) return 2;\n"
        '  if (strcmp(flxGetErrorString(flxInvalidArgument), "invalid argument")) return 3;\n'
        "  if (flxAllReduce(NULL, NULL, 1, flxFloat32, flxSum, NULL, 0) != flxInvalidArgument)"
        " return 4;\n"
        '  printf("ok\\n"); return 0;\n}\n')
    libdir = comm.library_path().parent
    exe = tmp_path / "caller"
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror",
                    f"-I{cuda_inc}", f"-I{ROOT / 'include'}", str(src), f"-L{libdir}",
                    "-lflexlink", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stdout)


def test_flx_shares_env_is_validated_at_init(lib, monkeypatch):
    # FLX_SHARES pins every bucket at comm creation (programs that only use the
    # NCCL names); a malformed value fails the init loudly, before any device work
    comms = (ctypes.c_void_p * 2)()
    lib.flxGetLastError.restype = ctypes.c_char_p
    for bad in ("900", "900,50", "a,b", "1000,0,0,0", "-5,1005", "900;100"):
        monkeypatch.setenv("FLX_SHARES", bad)
        assert lib.flxCommInitAll(comms, 2, None) == 4, bad
        assert b"FLX_SHARES" in lib.flxGetLastError(), bad


def test_shim_defines_every_communicator_call_pytorch_imports(lib):
    """Under LD_PRELOAD every NCCL call PyTorch's ProcessGroupNCCL can make with a
    communicator must resolve to the shim (implemented or refused): one that fell
    through to libnccl would get a FlexLink handle as its own struct.  Only the
    communicator-free calls may still resolve to NCCL."""
    import torch

    torch_cuda = Path(torch.__file__).parent / "lib" / "libtorch_cuda.so"
    shim = comm.library_path().parent / "libflexlink_nccl.so"
    if not torch_cuda.exists() or not shim.exists():
        pytest.skip("libtorch_cuda.so or the shim is absent")
    imported = {line.split()[-1] for line in subprocess.run(
        ["nm", "-D", str(torch_cuda)], capture_output=True, text=True, check=True).stdout
        .splitlines() if " U nccl" in line}
    defined = {line.split()[-1] for line in subprocess.run(
        ["nm", "-D", "--defined-only", str(shim)], capture_output=True, text=True,
        check=True).stdout.splitlines() if " T " in line}
    assert imported, "libtorch_cuda.so imports no NCCL symbols?"
    assert imported - defined <= {"ncclGroupSimulateEnd", "ncclMemAlloc", "ncclMemFree"}, \
        sorted(imported - defined)

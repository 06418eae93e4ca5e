"""NVLink-SHARP (multimem.ld_reduce / multimem.st) AllReduce, capability-gated.

flxNvlsProbe makes a one-device multicast object, binds and maps it, and runs
the NVLS kernel on it (ld_reduce over one rank is the identity), exact.  Where
the box cannot make multicast objects (a single-GPU lease outside an NVLink
fabric partition) the probe must say why, and the multi-GPU path stays on the
two-shot kernels; tools/nvls_diag.py records the fabric state beside it."""

import pytest

from paper_2510_15882_b200 import comm

pytestmark = pytest.mark.gpu


def test_nvls_probe_reports_capability_and_reason():
    ok, why = comm.nvls_probe(0)
    assert why, "the probe must explain its verdict"
    if not ok:
        pytest.skip(f"NVLS unavailable on this box: {why}")
    assert why.startswith("ok")


def test_single_gpu_comms_report_nvls_off_with_reason():
    with comm.Clique(2, device=0) as c:
        on, why = c.comms[0].nvls()
        assert not on and "multi-GPU" in why

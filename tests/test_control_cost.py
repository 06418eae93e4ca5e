"""SURVEY §8(d) control-plane timing: the library's balancer (flxTuneStep /
flxBalancerObserve, timed by tools/control_cost.c) and the reference algorithm's
Python (stage1 / stage2) take the same decisions on the same path-time model —
bench.py's `control_plane` block.  Host code only."""
import pytest


def test_native_and_python_balancers_agree_and_native_is_cheaper():
    from paper_2510_15882_b200 import comm

    try:
        comm.load_library()
    except Exception as e:  # the CPU suite builds the library first (test_library.py)
        pytest.skip(f"libflexlink.so not built: {e}")
    import bench

    r = bench.control_plane(target_s=0.2)
    assert r["decisions_agree"], r
    assert r["native"]["stage1_iterations"] > 3  # a real trajectory, not an instant stable
    assert r["native"]["stage2_moves"] > 0       # the PCIe shift is followed
    assert r["native"]["tune_step_ns"] < 1000 * r["reference_python"]["tune_step_us"]

"""The multi-rank PCIe path's constant-valued token handshake (csrc/world.cu
token_post / token_accept / token_give / take_region), model-checked with the
reference's interleaving explorer (staging.py:205-301, restated in pipeline.py):
every interleaving of producer and consumer reads the right iteration's data and
none deadlocks.  Its values never depend on the iteration, which is what lets a
CUDA graph replay the same stream memory operations."""

import pytest

from paper_2510_15882_b200.pipeline import explore_protocol, handshake_script


@pytest.mark.parametrize("iterations,buffers", [(1, 1), (2, 1), (4, 1), (6, 1), (4, 2), (6, 2)])
def test_token_handshake_has_no_stale_read_and_no_deadlock(iterations, buffers):
    v = explore_protocol(iterations, buffers, "token")
    assert v.ok and v.witness is None and v.deadlocks == 0


def test_token_values_are_iteration_independent():
    prod, cons = handshake_script(5, 1, "token")
    # the same four (kind, variable, value) steps every iteration: replayable
    per_iter = {tuple((k, var, arg) for k, var, _, arg, _ in prod[i * 4:(i + 1) * 4] if var != "buffer")
                for i in range(5)}
    assert len(per_iter) == 1
    per_iter = {tuple((k, var, arg) for k, var, _, arg, _ in cons[i * 4:(i + 1) * 4] if var != "buffer")
                for i in range(5)}
    assert len(per_iter) == 1


def test_reference_variants_unchanged():
    assert explore_protocol(4, 1, "counter").ok
    assert not explore_protocol(4, 1, "binary").ok
    with pytest.raises(ValueError):
        explore_protocol(2, 1, "nope")

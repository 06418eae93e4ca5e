"""Shared-interface bandwidth split and seeded run-to-run noise.

Restates the parts of the reference's ``linkstripe.simcore`` that the striped
collective and Stage 1 depend on (`pkg/src/linkstripe/simcore.py`):
:func:`maxmin_rates` (`simcore.py:100-130`), :func:`effective_bandwidths`
(`simcore.py:242-261`), :class:`NoiseModel` (`simcore.py:34-51`) and
:class:`SimClock` (`simcore.py:22-31`).  The fluid transfer engine
(`run_transfers`) is not on the collective path and is not rebuilt.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .links import PathKind, TopologySpec

__all__ = ["CONTENTION_GROUP", "SimClock", "NoiseModel", "maxmin_rates",
           "effective_bandwidths"]

# paths that leave the GPU through the same PCIe interface (`simcore.py:19`)
CONTENTION_GROUP = (PathKind.PCIE_STAGED, PathKind.RDMA_NIC)


class SimClock:
    """A clock that refuses to run backwards."""

    def __init__(self) -> None:
        self.now = 0.0

    def advance_to(self, t: float) -> None:
        if t < self.now:
            raise ValueError(f"clock moved backwards: {t} < {self.now}")
        self.now = t


@dataclass(frozen=True)
class NoiseModel:
    """Multiplicative per-path duration jitter, uniform on [1-sigma, 1+sigma]."""

    sigma: float = 0.0
    seed: int = 0

    def __post_init__(self) -> None:
        if not (0.0 <= self.sigma <= 0.5):
            raise ValueError("sigma must lie in [0, 0.5]")

    def stream(self) -> random.Random:
        return random.Random(self.seed)

    def factor(self, rng: random.Random) -> float:
        return 1.0 if self.sigma == 0.0 else rng.uniform(1.0 - self.sigma, 1.0 + self.sigma)


def maxmin_rates(demands: dict[int, float],
                 groups: list[tuple[set[int], float]]) -> dict[int, float]:
    """Progressive-filling max-min fair rates.

    Every flow is capped by its own demand and by each (members, capacity)
    group it belongs to.  All unfrozen flows rise at a common level; the
    tightest constraint freezes its members at that level, and so on.
    """
    rate = dict.fromkeys(demands, 0.0)
    done: set[int] = set()
    level = 0.0
    limits = [({flow}, cap) for flow, cap in demands.items()] + list(groups)
    while len(done) < len(rate):
        tightest = None
        for members, cap in limits:
            live = [f for f in members if f not in done]
            if not live:
                continue
            spent = sum(rate[f] for f in members if f in done)
            room = (cap - spent - level * len(live)) / len(live)
            if tightest is None or room < tightest[0]:
                tightest = (room, members)
        if tightest is None:
            break
        room, members = tightest
        level += max(room, 0.0)
        for f in members:
            if f not in done:
                rate[f] = level
                done.add(f)
    return rate


def effective_bandwidths(topo: TopologySpec, active_paths) -> dict[PathKind, float]:
    """Usable per-path rate while the given paths run at once.

    Without contention every path keeps its link rate; with it, the staged
    and NIC paths split ``shared_interface_bw`` max-min fairly.
    """
    paths = sorted(set(active_paths))
    rates = {p: topo.link(p).bandwidth_uni for p in paths}
    if not topo.path_contention:
        return rates
    sharing = [p for p in paths if p in CONTENTION_GROUP]
    if not sharing:
        return rates
    wants = {int(p): topo.link(p).bandwidth_uni for p in sharing}
    split = maxmin_rates(wants, [(set(wants), topo.shared_interface_bw)])
    for p in sharing:
        rates[p] = split[int(p)]
    return rates

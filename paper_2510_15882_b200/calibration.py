"""Alpha-beta calibration of the link profile from measured collective rows.

SURVEY §8(f) row 2.  The reference fits effective per-path parameters from a
table of measured end-to-end rows (`pkg/src/linkstripe/bench.py:111-227`,
``calibrate`` / ``build_calibrated_topology``) — its own table is the paper's
8xH800 Table 2 (`bench.py:72-106`).  Here the same fit runs
on either that table (golden-checked against the reference, tests/golden/
calibration.json) or on THIS run's measurements: ``bench.py`` sweeps the
NVLink-only collective over sizes (and NCCL beside it on N GPUs), fits
``1/algbw = a + b/size`` per (collective, N), and turns the balanced split the
in-library balancer settles on into the secondary paths' effective bandwidth —
a :class:`~paper_2510_15882_b200.links.TopologySpec` that ``set_link_profile``
hands to Stage 1 as its seed.

Model (the reference's ring model, collectives.py:136-186): a collective of
per-rank ``size`` bytes over ``n`` ranks runs ``steps = ring_steps(op, n)``
steps of ``size/n`` bytes, each costing ``size/(n*B) + L``, so

    1 / algbw = steps / (n * B) + steps * L / size        (algbw = size / t)

is linear in ``x = 1/size``: intercept ``a = steps/(n*B)``, slope ``b = steps*L``.
Secondary paths follow the balanced-completion identity: at the balancer's
split every path finishes together, so ``B_sec = B_nvlink * load_sec / load_nv``
(averaged over sizes with size weights — small sizes are latency-dominated).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .links import LinkSpec, PathKind, TopologySpec
from .striping import CollectiveOp, ring_steps

__all__ = ["MODE_BASELINE", "MODE_PCIE_ONLY", "MODE_PCIE_RDMA", "MODE_PATHS", "MeasuredRow",
           "LinkFit", "CalibrationResult", "CalibrationError", "H800_MEASUREMENTS",
           "fit_alpha_beta", "calibrate", "build_calibrated_topology", "CALIBRATED_CHUNK",
           "check_offload_identity", "ReproducedCell", "reproduce_reference",
           "check_reproduction", "EXPECTED_IDLE_PCT", "check_idle_goldens",
           "run_golden_checks"]

MODE_BASELINE = "nvlink_only"
MODE_PCIE_ONLY = "pcie_only"
MODE_PCIE_RDMA = "pcie_rdma"
MODE_PATHS = {
    MODE_BASELINE: (PathKind.NVLINK,),
    MODE_PCIE_ONLY: (PathKind.NVLINK, PathKind.PCIE_STAGED),
    MODE_PCIE_RDMA: (PathKind.NVLINK, PathKind.PCIE_STAGED, PathKind.RDMA_NIC),
}
MIB = 1 << 20
# staging chunk of a calibrated topology: small, so the pipeline fill the
# model adds stays negligible (the fitted bandwidth already includes staging)
CALIBRATED_CHUNK = 64 << 10


class CalibrationError(ValueError):
    """The rows do not admit a physical fit (the reference's CalibrationError)."""


@dataclass(frozen=True)
class MeasuredRow:
    """A measured row: algbw in GB/s, loads in percent of the message bytes."""

    op: CollectiveOp
    n_gpus: int
    size: int
    mode: str
    algbw: float
    impr_pct: int = 0
    pcie_load: float = 0.0
    rdma_load: float = 0.0

    @property
    def total_load(self) -> float:
        return self.pcie_load + self.rdma_load


@dataclass
class LinkFit:
    bandwidth: float  # B/s, effective per-direction link rate of the ring model
    latency: float    # s per ring step
    residuals: dict[int, float] = field(default_factory=dict)  # size -> (model-meas)/meas


@dataclass
class CalibrationResult:
    nvlink: dict[tuple[CollectiveOp, int], LinkFit]
    secondary: dict[tuple[CollectiveOp, int, str], dict[PathKind, float]]


# The paper's Table 2 (8xH800, NCCL 2.27.3 baseline), as the
# reference ships it (bench.py:72-106).  One line per (collective, N, MiB):
# NVLink-only GB/s | PCIe-only GB/s, gain %, PCIe load % | PCIe+RDMA GB/s,
# gain %, PCIe load %, RDMA load %.
_TABLE2 = """
allreduce 2  32 112 131 17 14 134 20 16  4
allreduce 2  64 128 144 13 17 150 17 13  5
allreduce 2 128 132 155 17 17 165 25 11  9
allreduce 2 256 139 167 20 18 175 26 12  9
allreduce 4  32  87  87  0  0  89  2  2  1
allreduce 4  64  90  97  8  8  99 10  6  2
allreduce 4 128  94 106 13 12 110 17 12  2
allreduce 4 256  98 116 18 17 118 20 13  5
allreduce 8 256 107 108  1  1 109  2  1  1
allgather 2  32 103 122 18 15 126 22 10  8
allgather 2  64 117 136 16 19 141 21  9 10
allgather 2 128 129 153 19 21 153 19 12  8
allgather 2 256 132 163 23 21 161 22 14  5
allgather 4  32  43  50 16 13  52 21 10  7
allgather 4  64  46  56 22 18  57 24 12  8
allgather 4 128  48  58 21 18  60 25 12 10
allgather 4 256  49  60 22 18  62 27 12 10
allgather 8  32  20  23 15 12  24 20 12  4
allgather 8  64  21  24 14 13  26 24 12  6
allgather 8 128  21  25 19 14  25 19 12  7
allgather 8 256  21  25 19 13  26 24 12  7
"""


def _parse_table2(text: str) -> tuple[MeasuredRow, ...]:
    rows: list[MeasuredRow] = []
    for line in text.strip().splitlines():
        name, *vals = line.split()
        op = CollectiveOp(name)
        n, mib, base, pb, pi, pl, rb, ri, rp, rr = (int(v) for v in vals)
        size = mib * MIB
        rows.append(MeasuredRow(op, n, size, MODE_BASELINE, base))
        rows.append(MeasuredRow(op, n, size, MODE_PCIE_ONLY, pb, pi, pl))
        rows.append(MeasuredRow(op, n, size, MODE_PCIE_RDMA, rb, ri, rp, rr))
    return tuple(rows)


H800_MEASUREMENTS: tuple[MeasuredRow, ...] = _parse_table2(_TABLE2)


def fit_alpha_beta(points: list[tuple[int, float]]) -> tuple[float, float]:
    """Ordinary least squares of ``y = 1/algbw`` on ``x = 1/size``.

    ``points`` are (size bytes, algbw B/s).  One point: pure bandwidth.  A
    negative slope (bandwidth rising slower than any latency explains) is
    folded into the intercept (mean of y), the residuals then show the misfit.
    Returns the intercept ``a`` and slope ``b``.
    """
    if not points:
        raise CalibrationError("no rows to fit")
    inv = [(1.0 / s, 1.0 / bw) for s, bw in points]
    if len(inv) == 1:
        return inv[0][1], 0.0
    n = len(inv)
    mx = sum(x for x, _ in inv) / n
    my = sum(y for _, y in inv) / n
    sxx = sum((x - mx) ** 2 for x, _ in inv)
    sxy = sum((x - mx) * (y - my) for x, y in inv)
    slope = sxy / sxx if sxx else 0.0
    if slope < 0:
        return my, 0.0
    return my - slope * mx, slope


def _group(rows, key):
    out: dict = {}
    for r in rows:
        out.setdefault(key(r), []).append(r)
    return out


def calibrate(rows) -> CalibrationResult:
    """Fit NVLink's (B, L) per (op, N) from the baseline rows, then every offload
    mode's secondary effective bandwidths from its load split."""
    base = _group([r for r in rows if r.mode == MODE_BASELINE], lambda r: (r.op, r.n_gpus))
    modes = _group([r for r in rows if r.mode != MODE_BASELINE],
                   lambda r: (r.op, r.n_gpus, r.mode))
    nvlink: dict[tuple[CollectiveOp, int], LinkFit] = {}
    for (op, n) in sorted(base, key=lambda k: (k[0].value, k[1])):
        pts = sorted((r.size, r.algbw * 1e9) for r in base[(op, n)])
        a, b = fit_alpha_beta(pts)
        if a <= 0:
            cells = ", ".join(f"{op.value}/{n}gpus/{s}B" for s, _ in pts)
            raise CalibrationError(f"infeasible bandwidth fit (a={a:.3e}) from rows: {cells}")
        steps = ring_steps(op, n)
        fit = LinkFit(bandwidth=steps / (n * a), latency=b / steps)
        fit.residuals = {s: ((1.0 / (a + b / s)) - bw) / bw for s, bw in pts}
        nvlink[(op, n)] = fit
    secondary: dict[tuple[CollectiveOp, int, str], dict[PathKind, float]] = {}
    for (op, n, mode) in sorted(modes, key=lambda k: (k[0].value, k[1], k[2])):
        anchor = nvlink.get((op, n))
        if anchor is None:
            raise CalibrationError(f"no baseline rows to anchor {op.value}/{n}gpus/{mode}")
        wsum = p_acc = r_acc = 0.0
        for r in modes[(op, n, mode)]:
            nv_part = 1.0 - r.total_load / 100.0
            if nv_part <= 0:
                raise CalibrationError(f"offload load is 100% in {op.value}/{n}gpus/{mode}")
            wsum += r.size
            p_acc += r.size * anchor.bandwidth * (r.pcie_load / 100.0) / nv_part
            r_acc += r.size * anchor.bandwidth * (r.rdma_load / 100.0) / nv_part
        fits = {PathKind.PCIE_STAGED: p_acc / wsum}
        if mode == MODE_PCIE_RDMA:
            fits[PathKind.RDMA_NIC] = r_acc / wsum
        secondary[(op, n, mode)] = fits
    return CalibrationResult(nvlink=nvlink, secondary=secondary)


def build_calibrated_topology(cal: CalibrationResult, op: CollectiveOp, n_gpus: int,
                              mode: str) -> TopologySpec:
    """A contention-free topology carrying the fitted parameters (contention and
    staging losses are inside the fitted rates), one per-step latency for all paths."""
    fit = cal.nvlink[(op, n_gpus)]
    links = {PathKind.NVLINK: LinkSpec(PathKind.NVLINK, fit.bandwidth, base_latency=fit.latency)}
    if mode != MODE_BASELINE:
        for kind, bw in cal.secondary[(op, n_gpus, mode)].items():
            links[kind] = LinkSpec(kind, bw, base_latency=fit.latency,
                                   staging_chunk=CALIBRATED_CHUNK)
    return TopologySpec(n_gpus=n_gpus, links=links, name=f"calibrated-{op.value}-{n_gpus}")


def check_offload_identity(rows=H800_MEASUREMENTS, size: int = 256 * MIB,
                           tolerance_pp: float = 5.0) -> list[str]:
    """At large sizes the gain should follow load/(1-load) (bench.py:365-380)."""
    bad = []
    for r in rows:
        if r.mode == MODE_BASELINE or r.size != size:
            continue
        load = r.total_load / 100.0
        want = 100.0 * load / (1.0 - load)
        if abs(r.impr_pct - want) > tolerance_pp:
            bad.append(f"{r.op.value}/{r.n_gpus}gpus/{r.mode}: improvement {r.impr_pct}% vs "
                       f"load identity {want:.1f}%")
    return bad


@dataclass
class ReproducedCell:
    """Calibrated-and-retuned simulation vs the published cell (bench.py:283-305)."""

    op: CollectiveOp
    n_gpus: int
    size: int
    mode: str
    published_bw: float
    simulated_bw: float
    published_offload: float
    simulated_offload: float
    baseline_residual: float

    @property
    def bw_rel_err(self) -> float:
        return (self.simulated_bw - self.published_bw) / self.published_bw

    @property
    def offload_err_pp(self) -> float:
        return self.simulated_offload - self.published_offload


def reproduce_reference(rows=H800_MEASUREMENTS, mode: str = MODE_PCIE_RDMA,
                        size: int = 256 * MIB, tuner=None) -> list[ReproducedCell]:
    """Calibrate from ``rows``, build each cell's topology, run Stage 1 on the
    model and compare with the published numbers (bench.py:318-355)."""
    from .stage1 import TunerConfig, initial_tune
    from .striping import CollectiveSpec, ShareDistribution, simulate_collective

    cal = calibrate(rows)
    out = []
    for r in rows:
        if r.mode != mode or r.size != size:
            continue
        topo = build_calibrated_topology(cal, r.op, r.n_gpus, mode)
        spec = CollectiveSpec(r.op, r.n_gpus, size)
        nv_only = topo.restricted(MODE_PATHS[MODE_BASELINE])
        simulate_collective(nv_only, spec, ShareDistribution({PathKind.NVLINK: 1000}))
        shares, _ = initial_tune(topo, spec, tuner or TunerConfig())
        rep = simulate_collective(topo, spec, shares)
        out.append(ReproducedCell(r.op, r.n_gpus, size, mode, r.algbw, rep.algbw / 1e9,
                                  r.total_load, (1000 - shares.get(PathKind.NVLINK)) / 10.0,
                                  cal.nvlink[(r.op, r.n_gpus)].residuals[size]))
    return out


def check_reproduction(bw_tolerance: float = 0.15, offload_tolerance_pp: float = 8.0) -> list[str]:
    """The calibrated model must land near the published table (bench.py:383-406)."""
    bad = []
    per_op: dict[CollectiveOp, dict[int, float]] = {}
    for c in reproduce_reference():
        per_op.setdefault(c.op, {})[c.n_gpus] = c.simulated_offload
        if abs(c.bw_rel_err) > bw_tolerance:
            bad.append(f"{c.op.value}/{c.n_gpus}gpus: simulated {c.simulated_bw:.1f} GB/s "
                       f"vs published {c.published_bw:.1f} ({c.bw_rel_err:+.1%})")
        if abs(c.offload_err_pp) > offload_tolerance_pp:
            bad.append(f"{c.op.value}/{c.n_gpus}gpus: simulated offload "
                       f"{c.simulated_offload:.1f}% vs published {c.published_offload:.1f}%")
    ar = per_op.get(CollectiveOp.ALLREDUCE, {})
    if ar and 8 in ar and any(ar[8] >= ar[k] for k in ar if k != 8):
        bad.append(f"8-GPU reduce offload {ar[8]:.1f}% is not the smallest of {ar}")
    return bad


# Idle-bandwidth headroom of each preset, percent of NVLink (bench.py:109; Table 1)
EXPECTED_IDLE_PCT = {"H800": 32, "H100": 14, "A800": 16, "GB200": 22, "GB300": 33}


def check_idle_goldens() -> list[str]:
    """Preset headroom vs the published Table-1 column (bench.py:357-363)."""
    from .links import idle_bw_opportunity, preset

    bad = []
    for name, want in EXPECTED_IDLE_PCT.items():
        got = round(idle_bw_opportunity(preset(name)) * 100)
        if got != want:
            bad.append(f"{name}: idle headroom {got}% != published {want}%")
    return bad


def run_golden_checks() -> list[str]:
    """Every golden comparison of the reference's harness (bench.py:409-414)."""
    return check_idle_goldens() + check_offload_identity() + check_reproduction()

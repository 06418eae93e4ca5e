"""FlexLink on B200: NCCL-shaped AllReduce/AllGather striped across NVLink,
host-staged PCIe and (when present) RDMA NICs, balanced by a two-stage tuner.

The names below mirror the reference package ``linkstripe``
(`pkg/src/linkstripe/__init__.py`) for the hot path — links, shares,
partition, timing reports, Stage 1 (``initial_tune``), Stage 2
(``run_dynamic`` & co.), the staging pipeline model and the optimum
references — so ``import paper_2510_15882_b200 as linkstripe`` works for that
surface.  The native data plane (``libflexlink.so``) is reached through
:mod:`paper_2510_15882_b200.comm`.
"""

from .calibration import (H800_MEASUREMENTS, CalibrationError, CalibrationResult, LinkFit,
                          MeasuredRow, build_calibrated_topology, calibrate)
from .fairshare import NoiseModel, SimClock, effective_bandwidths, maxmin_rates
from .links import (LinkSpec, PathKind, TopologySpec, idle_bw_opportunity, load_topology,
                    preset, topology_for)
from .optimum import OracleResult, closed_form_shares, optimal_shares_bruteforce
from .pipeline import (PipelineSpec, ProtocolVerdict, explore_protocol, pipeline_time,
                       simulate_pipeline_events)
from .stage1 import TunerConfig, TunerState, TuneTrace, initial_tune, initialize_shares, tune_step
from .stage2 import (Adjustment, BalancerConfig, BandwidthShift, DynamicResult, RuntimeBalancer,
                     TimingWindow, apply_adjustment, evaluate, median_durations, run_dynamic,
                     window_gap)
from .striping import (GRANULE_TOTAL, CollectiveOp, CollectiveSpec, PathTimingReport,
                       ShareDistribution, ShareTable, partition, ring_steps, simulate_collective,
                       size_bucket)
from .units import parse_bandwidth, parse_size, parse_time

__version__ = "1.0.0"

__all__ = [
    "H800_MEASUREMENTS", "CalibrationError", "CalibrationResult", "LinkFit", "MeasuredRow",
    "build_calibrated_topology", "calibrate",
    "Adjustment", "BalancerConfig", "BandwidthShift", "CollectiveOp", "CollectiveSpec",
    "DynamicResult", "GRANULE_TOTAL", "LinkSpec", "NoiseModel", "OracleResult", "PathKind",
    "PathTimingReport", "PipelineSpec", "ProtocolVerdict", "RuntimeBalancer", "ShareDistribution",
    "ShareTable", "SimClock", "TimingWindow", "TopologySpec", "TuneTrace", "TunerConfig",
    "TunerState", "apply_adjustment", "closed_form_shares", "effective_bandwidths", "evaluate",
    "explore_protocol", "idle_bw_opportunity", "initial_tune", "initialize_shares",
    "load_topology", "maxmin_rates", "median_durations", "optimal_shares_bruteforce",
    "parse_bandwidth", "parse_size", "parse_time", "partition", "pipeline_time", "preset",
    "ring_steps", "run_dynamic", "simulate_collective", "simulate_pipeline_events", "size_bucket",
    "topology_for", "tune_step", "window_gap",
]

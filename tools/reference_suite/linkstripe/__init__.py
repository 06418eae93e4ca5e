"""Alias package: the reference's module names (``linkstripe.topo``,
``linkstripe.collectives``, ...) bound to this repo's control plane, so the
reference's own test-suite runs against it (``tools/reference_suite/run.py``,
``tests/test_reference_suite.py``).  Test infrastructure only — never
installed, never imported by the product.

Modules the tier framing leaves out of scope (the reference CLI ``cli.py``,
the simulated bench-table generator in ``bench.py`` — its calibration IS
bound, to ``calibration.py`` — and the fluid transfer engine
``simcore.run_transfers``) are stubs whose callables raise
``NotImplementedError``: the tests that need them fail, and the runner lists
exactly which.
"""

import importlib
import sys
import types

from paper_2510_15882_b200 import *  # noqa: F401,F403

_MODULES = {
    "topo": "links",           # PathKind, LinkSpec, TopologySpec, preset, load_topology
    "collectives": "striping",  # ShareDistribution, partition, simulate_collective, ...
    "tuner": "stage1",          # initialize_shares, tune_step, initial_tune, write_trace
    "balancer": "stage2",       # TimingWindow, evaluate, run_dynamic, ...
    "staging": "pipeline",      # PipelineSpec, pipeline_time, explore_protocol
    "oracle": "optimum",        # closed_form_shares, optimal_shares_bruteforce
    "units": "units",
}
for _name, _ours in _MODULES.items():
    sys.modules[f"{__name__}.{_name}"] = importlib.import_module(f"paper_2510_15882_b200.{_ours}")


def _out_of_scope(what):
    def fn(*args, **kwargs):
        raise NotImplementedError(f"{what} is out of scope for this build (DESIGN.md §1)")
    fn.__name__ = what
    return fn


def _module(name, base=None, stubs=(), values=None):
    mod = types.ModuleType(f"{__name__}.{name}")
    if base is not None:
        mod.__dict__.update({k: v for k, v in vars(base).items() if not k.startswith("__")})
    for stub in stubs:
        setattr(mod, stub, _out_of_scope(f"linkstripe.{name}.{stub}"))
    for key, value in (values or {}).items():
        setattr(mod, key, value)
    sys.modules[mod.__name__] = mod
    return mod


# simcore: the max-min fair share (in scope, fairshare.py) + the fluid engine (out)
simcore = _module("simcore", importlib.import_module("paper_2510_15882_b200.fairshare"),
                  stubs=("TransferRequest", "run_transfers", "write_event_log"))
# bench.py: the calibration (calibration.py) is in scope; the simulated bench
# table generator and its formatting are not
bench = _module("bench", importlib.import_module("paper_2510_15882_b200.calibration"),
                stubs=("BenchPlan", "run_bench", "format_rows"))
# cli.py (out of scope)
cli = _module("cli", stubs=("main",))

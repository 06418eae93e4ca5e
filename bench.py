#!/usr/bin/env python
"""FlexLink-on-B200 benchmark: striped AllReduce/AllGather bus bandwidth.

Metric (BASELINE.json): AllReduce/AllGather busBW GB/s @256MB vs NCCL, plus the
PCIe/NIC traffic share.

* N=1 (default, ``python bench.py``): BASELINE config 1 — AllReduce sum fp32,
  256 MiB per rank over 8 simulated ranks — run as 8 *virtual ranks* on cuda:0
  (flxCommInitAll with a repeated device; one fused NVLink-path launch per call,
  the PCIe share through the real host-staged copy-engine pipeline).  Shares
  come from Stage 1 run on the real path (guarded), then a short Stage-2 phase.
  The AllGather bf16 256 MiB (config 2 shape, 8 virtual ranks) is reported in
  the same line under "allgather".
* N>1 (torchrun, one process per GPU): the same AllReduce, 256 MiB per rank,
  over N real GPUs through flxCommInitRank, with torch.distributed NCCL timed
  on the same buffers for the "nccl" column.
* ``--impl reference``: the reference's CPU path — the oracle port
  (oracle/flx_oracle.c, all host threads) on a bounded sample of the same
  workload.

busbw (nccl-tests): AllReduce (S/t)*2(N-1)/N, AllGather (S_out/t)*(N-1)/N.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MIB = 1 << 20
SIM_RANKS = 8
AR_BYTES = 256 * MIB           # per rank (config 1)
AG_OUT_BYTES = 256 * MIB       # gathered output (config 2, nccl-tests convention)
METRIC = "AllReduce/AllGather busBW GB/s @256MB vs NCCL; PCIe/NIC traffic share %"


# The JSON line goes to the process's original stdout; everything else the
# native libraries print (e.g. NCCL's "NCCL version ..." banner under torchrun)
# is routed to stderr, so rank 0's stdout is exactly ONE JSON line.
_JSON_FD: int | None = None


def emit(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def route_native_stdout_to_stderr() -> None:
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def busbw_allreduce(nbytes: int, seconds: float, n: int) -> float:
    return nbytes / seconds * 2 * (n - 1) / n / 1e9


def busbw_allgather(out_bytes: int, seconds: float, n: int) -> float:
    return out_bytes / seconds * (n - 1) / n / 1e9


PCIE_H2D_GBS = 55.5  # measured pinned H2D on this pool (profiles/r1/pcie_bidir.json)


def link_roofline(busbw: float, pcie_gbs: float | None) -> dict:
    """The north star's aggregate-link roofline: 900 GB/s/dir NVLink 5 + measured PCIe
    Gen5 + NIC (absent)."""
    pcie = round(pcie_gbs if pcie_gbs else PCIE_H2D_GBS, 1)
    peak = 900.0 + pcie
    return {"nvlink_gbs": 900.0, "pcie_gbs": pcie, "nic_gbs": 0.0, "peak": round(peak, 1),
            "achieved": round(busbw, 2), "frac": round(busbw / peak, 4)}


def ncu_traffic(summary: str = "profiles/r2/fold_once_ncu_summary.txt"):
    """dram read + write bytes per launch of the dominant kernel, from the
    committed ``ncu --set full`` capture of the same workload (None if absent)."""
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    try:
        with open(os.path.join(ROOT, summary)) as f:
            for line in f:
                parts = line.split()
                if len(parts) == 3 and parts[0] in ("dram__bytes_read.sum",
                                                    "dram__bytes_write.sum"):
                    total += float(parts[1]) * units[parts[2]]
    except (OSError, KeyError, ValueError):
        return None
    return int(total) if total else None


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons polled through NVML during the timed region
    (the B200_PROFILING.md clocks line, without nvidia-smi's startup latency)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, cuda_index: int = 0, period_s: float = 0.002):
        self.cuda_index = cuda_index
        self.period = period_s
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None
        self.error = None

    def start(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            idx = self.cuda_index
            try:
                idx = torch.cuda._get_nvml_device_index(self.cuda_index)
            except Exception:
                pass
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report it instead of guessing
            self.error = f"nvml unavailable: {e}"
            return self
        self.thread = threading.Thread(target=self._poll, daemon=True)
        self.thread.start()
        time.sleep(0.02)
        self.t0 = time.perf_counter()
        return self

    def _poll(self):
        n, h = self.nvml, self.handle
        while not self._stop.is_set():
            try:
                mhz = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
                why = n.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((mhz, why))
            except Exception as e:
                self.error = str(e)
                return
            time.sleep(self.period)

    def stop(self) -> dict:
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [],
                    "samples": 0, "note": self.error or "no samples"}
        reasons = set()
        for _, why in self.samples:
            for bit, name in self.REASONS.items():
                if why & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(m for m, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(self.samples),
                # the sampled window (NVML polls every 2 ms, slower when NVML is slow)
                "window_ms": round((time.perf_counter() - getattr(self, "t0", 0.0)) * 1e3, 1)}


def workload_config(n_gpus: int) -> dict:
    """The ``config`` both arms report (the reference arm samples it on the host)."""
    if n_gpus > 1:
        return {"workload": f"AllReduce sum fp32 256 MiB/rank over {n_gpus} GPUs",
                "bytes_per_rank": AR_BYTES}
    return {"workload": "AllReduce sum fp32 256 MiB/rank over 8 simulated ranks (BASELINE "
                        "config 1) as 8 virtual ranks on one B200; NVLink path = fused "
                        "on-device fold, PCIe path = real host-staged copy-engine pipeline",
            "sim_ranks": SIM_RANKS, "bytes_per_rank": AR_BYTES}


# ------------------------------------------------------------ CPU baseline
def cpu_model() -> str:
    """Host CPU model and logical CPU count (printed with every CPU timing)."""
    name = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                name = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{name}, {os.cpu_count()} logical CPUs"


def cpu_allreduce_sample(target_s: float = 10.0, per_rank_bytes: int = AR_BYTES,
                         n: int = SIM_RANKS):
    """Oracle port on the host: the same n-rank fp32 AllReduce (256 MiB per rank)
    repeated until ~target_s."""
    import numpy as np

    import oracle

    oracle.build()
    threads = oracle.cpu_threads()
    count = per_rank_bytes // 4
    rng = np.random.default_rng(1000)
    sends = [rng.integers(-1024, 1024, count).astype(np.float32) for _ in range(n)]
    recvs = [np.zeros_like(s) for s in sends]  # pre-touched: no page faults in the timing
    oracle.allreduce(sends, 7, oracle.SUM, recvs=recvs, threads=threads)  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.allreduce(sends, 7, oracle.SUM, recvs=recvs, threads=threads)
        reps += 1
        if time.perf_counter() - t0 >= target_s:
            break
    per_call = (time.perf_counter() - t0) / reps
    return {
        "value": round(busbw_allreduce(per_rank_bytes, per_call, n), 3),
        "unit": "GB/s",
        "cores": threads,
        "kind": "port",
        "cpu": cpu_model(),
        "sample": f"AllReduce sum fp32 {per_rank_bytes // MIB} MiB/rank x {n} simulated ranks, "
                  f"{reps} calls in {per_call * reps:.1f} s (oracle/flx_oracle.c, OpenMP)",
    }


def control_plane(target_s: float = 1.0) -> dict:
    """SURVEY §8(d) CPU-path timing of the control plane: the balancer's decisions in
    the reference algorithm's own Python (stage1 / stage2, restating tuner.py:134-226
    and balancer.py:57-207; 1 core) beside the library's C++ (flxTuneStep /
    flxBalancerObserve, tools/control_cost.c), both driven by one closed-form
    path-time model — Stage 1 from the H800 three-path profile with observed rates
    below it, then 1000 Stage-2 calls with PCIe at 0.7x from call 31.  The two must
    take the same decisions (iterations and final shares)."""
    import subprocess

    from paper_2510_15882_b200 import links, stage1, stage2, striping
    from paper_2510_15882_b200.links import PathKind

    root = os.path.dirname(os.path.abspath(__file__))
    exe = os.path.join(root, "tools", "bin", "control_cost")
    src = os.path.join(root, "tools", "control_cost.c")
    lib = os.path.join(root, "paper_2510_15882_b200")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(exe), exist_ok=True)
        subprocess.run(["gcc", "-O2", "-I", os.path.join(root, "include"), "-I",
                        "/usr/local/cuda/include", src, "-L", lib, "-lflexlink",
                        f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    native = json.loads(subprocess.run([exe], check=True, capture_output=True,
                                       text=True).stdout)

    topo = links.preset("H800")
    lat = {PathKind.NVLINK: 5e-6, PathKind.PCIE_STAGED: 1e-5, PathKind.RDMA_NIC: 1.5e-5}
    obs = {PathKind.NVLINK: 190e9, PathKind.PCIE_STAGED: 40e9, PathKind.RDMA_NIC: 6.25e9}
    size = 256 * MIB
    moved = float(size) * 2.0 * 7.0 / 8.0
    spec = striping.CollectiveSpec(striping.CollectiveOp.ALLREDUCE, 8, size)

    def model(shares, active, scale=1.0):
        d = {p: lat[p] + (moved * shares.get(p) / 1000.0) /
             (obs[p] * scale if p == PathKind.PCIE_STAGED else obs[p]) for p in active}
        return striping.PathTimingReport.build(spec.op, spec.n_gpus, spec.size, d)

    def tune():
        return stage1.initial_tune(topo, spec, measure=lambda st: model(st.shares, st.active))

    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < target_s:
        shares, trace = tune()
        reps += 1
    s1 = (time.perf_counter() - t0) / reps
    iters = len(trace.records)
    active = shares.loaded_paths

    def dynamic():
        return stage2.run_dynamic(
            topo, spec, shares, n_calls=1000, active=active,
            measure=lambda call, sh: model(sh, active, 0.7 if call >= 31 else 1.0))

    # observe() alone: replay the reports of one run through a fresh hook
    res = dynamic()
    reps2, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < target_s:
        hook = stage2.RuntimeBalancer(shares, active=active)
        for rep in res.reports:
            hook.observe(rep)
        reps2 += 1
    obs_us = (time.perf_counter() - t0) / (reps2 * len(res.reports)) * 1e6
    t0 = time.perf_counter()
    dynamic()
    dyn_ms = (time.perf_counter() - t0) * 1e3
    py = {"stage1_ms": round(s1 * 1e3, 4), "stage1_iterations": iters,
          "tune_step_us": round(s1 / max(iters, 1) * 1e6, 2),
          "stage1_shares": [shares.get(p) for p in PathKind],
          "observe_us": round(obs_us, 2),
          "run_dynamic_ms_per_1000_calls": round(dyn_ms, 2),
          "stage2_evaluations": len(res.evaluations),
          "stage2_moves": sum(1 for e in res.evaluations if e.adjustment is not None),
          "stage2_shares": [res.final_shares.get(p) for p in PathKind]}
    agree = all(native[k] == py[k] for k in ("stage1_iterations", "stage1_shares",
                                              "stage2_evaluations", "stage2_moves",
                                              "stage2_shares"))
    return {"reference_python": py, "native": native, "decisions_agree": agree,
            "speedup_tune_step": round(py["tune_step_us"] * 1e3 / native["tune_step_ns"], 1),
            "speedup_observe": round(py["observe_us"] * 1e3 / native["observe_ns"], 1),
            "cores": 1, "cpu": cpu_model(),
            "note": "per-decision host cost; the reference's Python is the restated "
                    "stage1/stage2 (tests/test_reference_suite.py passes the reference's own "
                    "tests against it); run_dynamic includes the model evaluation"}


def run_reference(args) -> None:
    """``--impl reference``: the CPU path on the box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import oracle

    oracle.build()
    threads = oracle.cpu_threads()
    per_rank = AR_BYTES  # the GPU arm's workload itself (same_config), not a sample
    count = per_rank // 4
    ranks = args.gpus if args.gpus > 1 else SIM_RANKS
    rng = np.random.default_rng(1000)
    sends = [rng.integers(-1024, 1024, count).astype(np.float32) for _ in range(ranks)]
    recvs = [np.zeros_like(s) for s in sends]  # pre-touched: no page faults in the timing
    for _ in range(max(args.warmup, 3)):  # OpenMP pool spin-up + caches
        oracle.allreduce(sends, 7, oracle.SUM, recvs=recvs, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.allreduce(sends, 7, oracle.SUM, recvs=recvs, threads=threads)
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    value = busbw_allreduce(per_rank, dt, ranks)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.gpus),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads,
                         "kind": "port", "cpu": cpu_model(),
                         "sample": f"each step: the full workload, AllReduce sum fp32 "
                                   f"{per_rank // MIB} MiB/rank x {ranks} ranks on the host "
                                   f"(oracle/flx_oracle.c, OpenMP, {threads} threads)"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


# --------------------------------------------------------------- N = 1
def _time_steps(fn, steps: int, stream) -> float:
    import torch

    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for _ in range(steps):
        fn()
    end.record(stream)
    torch.cuda.synchronize()
    return start.elapsed_time(end) / 1e3 / steps


def run_single_gpu(args) -> None:
    import torch

    from paper_2510_15882_b200 import comm as flx
    from paper_2510_15882_b200.links import PathKind, preset
    from paper_2510_15882_b200.striping import CollectiveOp, ShareDistribution

    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    n = SIM_RANKS
    count = AR_BYTES // 4
    gen = torch.Generator(device="cuda").manual_seed(1000)
    sends = [torch.randint(-1024, 1024, (count,), device="cuda", generator=gen).float()
             for _ in range(n)]
    recvs = [torch.empty_like(s) for s in sends]
    stream = torch.cuda.current_stream()
    clique = flx.Clique(n, device=0)
    if args.nvlink_ctas:
        clique.set_nvlink_ctas(args.nvlink_ctas)
    # Stage 1 seeds from MEASURED per-link bandwidth (probe), not a datasheet
    from paper_2510_15882_b200.probe import probe_topology, topology_to_yaml

    try:
        topo, probe_raw = probe_topology(nranks=n, name="probed-b200-virtual8")
        link_profile = {"yaml": topology_to_yaml(topo), "raw": probe_raw}
        link_bidir = probe_raw["pcie"]["bidir_each"]  # B/s per direction, both busy
        pcie_h2d = probe_raw["pcie"]["h2d"] / 1e9
    except Exception as e:  # keep the bench alive; fall back to the nominal preset
        link_bidir = pcie_h2d = None
        topo = preset("B200").restricted([PathKind.NVLINK, PathKind.PCIE_STAGED])
        link_profile = {"error": str(e), "fallback": "preset B200"}

    # ---- the in-library balancer (csrc/autotune.cpp): the bucket's first calls
    # run Stage 1 (NVLink-only baseline, measured-rate seed, Algorithm 1, guard),
    # every later call feeds Stage 2 — no flxSetShares, exactly what an
    # NCCL-API caller gets
    t0 = time.perf_counter()
    tune_calls = settle(clique, lambda: clique.all_reduce(sends, recvs), CollectiveOp.ALLREDUCE,
                        AR_BYTES)
    tune_wall = time.perf_counter() - t0
    tinfo = clique.tune_info(CollectiveOp.ALLREDUCE, AR_BYTES)
    trace = clique.tune_trace(CollectiveOp.ALLREDUCE, AR_BYTES)
    shares = ShareDistribution({k: tinfo["shares"][int(k)] for k in PathKind
                                if tinfo["shares"][int(k)] or k == PathKind.NVLINK})
    # the reference's closed-form model (simulate_collective, collectives.py:136-186) on
    # the probed link profile, for the split that runs: predicted vs measured per path
    from paper_2510_15882_b200.striping import CollectiveSpec, simulate_collective

    pred = simulate_collective(topo, CollectiveSpec(CollectiveOp.ALLREDUCE, n, AR_BYTES), shares,
                               alignment=clique.comms[0].alignment(CollectiveOp.ALLREDUCE))
    model_ms = {k.short: round(v * 1e3, 4) for k, v in pred.durations.items()}

    def step():
        clique.all_reduce(sends, recvs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(0).start()
    launches0 = flx.launch_count()
    dt = _time_steps(step, args.steps, stream)
    launches = flx.launch_count() - launches0
    clocks = sampler.stop()
    hist = clique.comms[0].path_times_history(min(args.steps, 64))
    pbytes = clique.path_bytes()
    nv_ms = statistics.mean(h[PathKind.NVLINK] for h in hist) * 1e3
    pc_ms = statistics.mean(h[PathKind.PCIE_STAGED] for h in hist) * 1e3 \
        if pbytes[PathKind.PCIE_STAGED] else 0.0
    value = busbw_allreduce(AR_BYTES, dt, n)
    nv_alg_bytes = 2 * n * pbytes[PathKind.NVLINK]  # N reads + N writes of the NVLink slice
    achieved = nv_alg_bytes / (nv_ms * 1e-3) / 1e9

    # library baseline on the same GPU: the same 8-rank AllReduce as unfused torch
    # ops (left fold with torch.add, then 8 copies) — what one GPU does without
    # the fused kernel (NCCL cannot run 8 ranks on one GPU)
    def torch_unfused():
        acc = torch.add(sends[0], sends[1])
        for s in sends[2:]:
            acc.add_(s)
        for r in recvs:
            r.copy_(acc)

    for _ in range(2):  # warm: allocator, kernels
        torch_unfused()
    torch_dt = _time_steps(torch_unfused, max(5, args.steps // 2), stream)
    torch_base = {"value": round(busbw_allreduce(AR_BYTES, torch_dt, n), 2),
                  "ms_per_step": round(torch_dt * 1e3, 4),
                  "what": "torch.add left fold + 8 copy_ (unfused, same GPU, same data)"}

    # exactness spot check of the timed result (integer-valued inputs: exact sum)
    exact = torch.stack(sends).sum(0)
    assert all(torch.equal(r, exact) for r in recvs), "allreduce result mismatch"

    # ---- e2e through the public API with host buffers
    host_in = [torch.empty(count, dtype=torch.float32, pin_memory=True) for _ in range(n)]
    # the reduced tensor comes back once: every virtual rank's recv holds the
    # same bytes (on N GPUs each rank reads its own copy over its own link)
    host_out = [torch.empty(count, dtype=torch.float32, pin_memory=True)]
    for h, s in zip(host_in, sends):
        h.copy_(s)

    # Two device buffer sets, in-place AllReduce: step k's D2H (on its own
    # stream) overlaps step k+1's H2D, using both PCIe directions at once.
    bufs = [sends, recvs]
    up = torch.cuda.Stream()
    down = torch.cuda.Stream()
    done_up = [torch.cuda.Event(), torch.cuda.Event()]
    done_ar = [torch.cuda.Event(), torch.cuda.Event()]
    done_down = [torch.cuda.Event(), torch.cuda.Event()]
    k_box = [0]

    def e2e_step():
        k = k_box[0] % 2
        k_box[0] += 1
        b = bufs[k]
        up.wait_event(done_down[k])            # buffer set k drained by its last D2H
        with torch.cuda.stream(up):
            for h, s in zip(host_in, b):
                s.copy_(h, non_blocking=True)
            done_up[k].record(up)
        stream.wait_event(done_up[k])
        clique.all_reduce(b, b)                # in place, public API
        done_ar[k].record(stream)
        down.wait_event(done_ar[k])
        with torch.cuda.stream(down):
            for h, r in zip(host_out, b):
                h.copy_(r, non_blocking=True)
            done_down[k].record(down)
        stream.wait_event(done_down[k])        # the step ends with its result on the host

    for _ in range(2):
        e2e_step()
    # the pipeline fills (first H2D alone) and drains (last D2H alone) once per
    # timed region: enough steps that the overlapped steady state dominates
    e2e_steps = max(3, min(args.steps, 40))
    e2e_dt = _time_steps(e2e_step, e2e_steps, stream)
    e2e_value = busbw_allreduce(AR_BYTES, e2e_dt, n)
    assert all(torch.equal(h, exact.cpu()) for h in host_out[:1]), "e2e result mismatch"
    for h, s in zip(host_in, sends):  # the e2e loop reduced in place: restore the inputs
        s.copy_(h)
    torch.cuda.synchronize()

    # ---- AllGather bf16, 256 MiB gathered (config 2 shape) over 8 virtual ranks
    ag_count = AG_OUT_BYTES // 2 // n
    ag_send = [torch.randn(ag_count, device="cuda", generator=gen).bfloat16() for _ in range(n)]
    ag_recv = [torch.empty(ag_count * n, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    settle(clique, lambda: clique.all_gather(ag_send, ag_recv), CollectiveOp.ALLGATHER,
           AG_OUT_BYTES // n)
    ag_info = clique.tune_info(CollectiveOp.ALLGATHER, AG_OUT_BYTES // n)
    ag_shares = ShareDistribution({k: ag_info["shares"][int(k)] for k in PathKind
                                   if ag_info["shares"][int(k)] or k == PathKind.NVLINK})
    for _ in range(args.warmup):
        clique.all_gather(ag_send, ag_recv)
    ag_dt = _time_steps(lambda: clique.all_gather(ag_send, ag_recv), args.steps, stream)
    ag_bytes = clique.path_bytes()
    ag_hist = clique.comms[0].path_times_history(min(args.steps, 64))
    ag_nv_ms = statistics.mean(h[PathKind.NVLINK] for h in ag_hist) * 1e3
    ag_alg = (n + n * n) * ag_bytes[PathKind.NVLINK]  # N reads + N^2 writes
    for r in range(n):
        for q in range(n):
            assert torch.equal(ag_recv[r][q * ag_count:(q + 1) * ag_count], ag_send[q])

    del ag_send, ag_recv

    # ---- ReduceScatter / AllToAll fp32 on the same 8 x 256 MiB inputs
    blk = count // n
    extra = {}
    rs_recv = [torch.empty(blk, device="cuda") for _ in range(n)]
    a2a_recv = [torch.empty_like(x) for x in sends]
    for name, cop, run, alg in (
            ("reducescatter", CollectiveOp.REDUCESCATTER,
             lambda: clique.reduce_scatter(sends, rs_recv), (n + 1) * AR_BYTES),
            ("alltoall", CollectiveOp.ALLTOALL, lambda: clique.all_to_all(sends, a2a_recv),
             2 * n * AR_BYTES)):
        # the library balances these buckets too (per-rank message = one block
        # of AR_BYTES / n): let it settle before timing
        tuned = settle(clique, run, cop, AR_BYTES // n)
        for _ in range(args.warmup):
            run()
        dt_c = _time_steps(run, args.steps, stream)
        hist = clique.comms[0].path_times_history(min(args.steps, 64))
        k_ms = statistics.mean(h[PathKind.NVLINK] for h in hist) * 1e3
        extra[name] = {"value": round(AR_BYTES / dt_c * (n - 1) / n / 1e9, 2), "unit": "GB/s",
                       "balancer": {"tuning_calls": tuned,
                                    **{k: v for k, v in clique.tune_info(cop, AR_BYTES // n).items()
                                       if k in ("phase", "kept_tuned", "shares")}},
                       "dtype": "f32", "send_bytes_per_rank": AR_BYTES,
                       "ms_per_step": round(dt_c * 1e3, 4),
                       "busbw": "(S_send/t)*(N-1)/N (nccl-tests)",
                       "kernel_algorithmic_bytes": alg,
                       "kernel_frac_hbm": round(alg / (k_ms * 1e-3) / 1e9 / hbm_peak, 4),
                       "traffic_share_pct": {k.short: round(100 * v / max(1, sum(
                           clique.path_bytes().values())), 3)
                                             for k, v in clique.path_bytes().items()},
                       "link_roofline": link_roofline(AR_BYTES / dt_c * (n - 1) / n / 1e9,
                                                      pcie_h2d)}
    for r in range(n):
        assert torch.equal(rs_recv[r], exact[r * blk:(r + 1) * blk]), "reduce_scatter mismatch"
        for q in range(n):
            assert torch.equal(a2a_recv[r][q * blk:(q + 1) * blk],
                               sends[q][r * blk:(r + 1) * blk]), "all_to_all mismatch"
    del rs_recv, a2a_recv

    cfg4 = run_config4(clique, sends, recvs, topo, args, stream) if not args.skip_config4 else None
    cfg5 = run_config5(clique, topo, stream) if not args.skip_config5 else None

    # ---- the multi-GPU engine (flxCommInitRank code path) emulated on this GPU
    loop = flx.Clique(n, device=0, loopback=True)
    loop.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
    for _ in range(2):
        loop.all_reduce(sends, recvs)
    loop_dt = _time_steps(lambda: loop.all_reduce(sends, recvs), args.steps, stream)
    assert all(torch.equal(r, exact) for r in recvs), "loopback allreduce mismatch"
    loop.set_shares(CollectiveOp.ALLREDUCE, (990, 10, 0))
    loop.all_reduce(sends, recvs)
    torch.cuda.synchronize()
    assert all(torch.equal(r, exact) for r in recvs), "loopback striped allreduce mismatch"
    loop_alg = int(n * (5 - 2 / n) * AR_BYTES)  # push 2(n-1)/n S + fold (1+2/n) S + pull 2(n-1)/n S
    loopback = {"busbw": round(busbw_allreduce(AR_BYTES, loop_dt, n), 2),
                "ms_per_step": round(loop_dt * 1e3, 4),
                "hbm_algorithmic_bytes": loop_alg,
                "hbm_frac": round(loop_alg / loop_dt / 1e9 / hbm_peak, 4),
                "note": "8 ranks of the one-process-per-GPU engine sharing one GPU's HBM "
                        "(push/reduce/pull through peer-mapped scratch; 3 HBM passes)"}
    loop.destroy()
    cpu = cpu_allreduce_sample(args.cpu_seconds)
    total = AR_BYTES
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded integer-valued fp32, exact-sum checked)",
        "config": {
            **workload_config(1), "busbw": "(S/t)*2(N-1)/N, N=8",
            "l2": "inputs 2 GiB + outputs 2 GiB per step > 126 MB L2 (no flush needed)",
            "nvlink_ctas": args.nvlink_ctas or "auto",
        },
        "shares": {k.short: shares.get(k) for k in PathKind},
        "path_bytes": {k.short: pbytes[k] for k in PathKind},
        "traffic_share_pct": {k.short: round(100 * pbytes[k] / total, 3) for k in PathKind},
        "path_ms": {"nvlink": round(nv_ms, 4), "pcie": round(pc_ms, 4), "rdma": None},
        "model_path_ms": {**model_ms, "source": "linkstripe simulate_collective on the probed "
                                                "link profile (the reference's predictor)"},
        "rdma": "absent (no NIC / rdma-core in this image)",
        "balancer": {"where": "in-library (csrc/autotune.cpp): Stage 1 + guard on the "
                              "bucket's first calls, Stage 2 on every call",
                     "tuning_calls": tune_calls, "tuning_wall_s": round(tune_wall, 2),
                     **tinfo, "stage1_trace": [r["action"] for r in trace]},
        "roofline": {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4),
            # the capture is of the full 256 MiB slice; another split has no capture
            "traffic": ncu_traffic() if pbytes[PathKind.NVLINK] == AR_BYTES else None,
            "traffic_source": "profiles/r2/fold_once_ncu_summary.txt (ncu --set full, same "
                              "kernel and size; dram__bytes_read.sum + dram__bytes_write.sum)",
            "kernel": "fold_once_kernel<float,Sum,8,1024> (NVLink-path slice, 8 virtual ranks, "
                      "one 16 B vector per thread)",
            "algorithmic_bytes_per_launch": nv_alg_bytes,
            "kernel_ms": round(nv_ms, 4),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
        },
        "link_roofline": {**link_roofline(value, pcie_h2d), "note": "at N=1 the NVLink path is "
                          "an on-GPU fold bound by HBM (see roofline); this is the north star's "
                          "multi-GPU denominator"},
        "cpu_baseline": cpu,
        "control_plane": control_plane(),
        "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                "h2d_bytes_per_step": n * AR_BYTES, "d2h_bytes_per_step": AR_BYTES,
                "ms_per_step": round(e2e_dt * 1e3, 3), "steps": e2e_steps,
                "link_bound_ms": round(n * AR_BYTES / (pcie_h2d * 1e9) * 1e3, 3) if pcie_h2d
                else None,
                "note": "all 8 ranks' inputs (2 GiB) in over ONE PCIe link per step and the "
                        "reduced tensor (identical in every virtual rank's recv) out once; "
                        "in-place AllReduce, step k's D2H overlapped with step k+1's H2D; "
                        "link_bound_ms = 2 GiB H2D at the probed H2D rate"},
        "gpu_launches": launches,
        "clocks": clocks,
        "nccl": None,
        "nccl_note": "NCCL cannot place 8 ranks on one GPU (duplicate device); the N>1 line "
                     "(torchrun, one process per GPU) times NCCL on the same box",
        "torch_unfused_baseline": torch_base,
        "link_profile": link_profile,
        "config4": cfg4,
        "config5": cfg5,
        "loopback_engine": loopback,
        **extra,
        "allgather": {
            "value": round(busbw_allgather(AG_OUT_BYTES, ag_dt, n), 2), "unit": "GB/s",
            "dtype": "bf16", "out_bytes": AG_OUT_BYTES, "ms_per_step": round(ag_dt * 1e3, 4),
            "shares": {k.short: ag_shares.get(k) for k in PathKind},
            "traffic_share_pct": {k.short: round(100 * ag_bytes[k] / (AG_OUT_BYTES // n), 3)
                                  for k in PathKind},
            "kernel_achieved_gbs": round(ag_alg / (ag_nv_ms * 1e-3) / 1e9, 1),
            "kernel_frac_hbm": round(ag_alg / (ag_nv_ms * 1e-3) / 1e9 / hbm_peak, 4),
            "kernel_algorithmic_bytes": ag_alg,
            "kernel_traffic": ncu_traffic("profiles/r1/fanout_once_ncu_summary.txt"),
            "paper_convention_algbw": round(AG_OUT_BYTES / n / ag_dt / 1e9, 2),
            "link_roofline": link_roofline(busbw_allgather(AG_OUT_BYTES, ag_dt, n), pcie_h2d),
        },
    }
    clique.destroy()
    emit(line)


def settle(clique, call, op, nbytes: int, limit: int = 400) -> int:
    """Issue ``call`` until the in-library balancer has left Stage 1 for the
    bucket (Stage 2 running), at most ``limit`` calls; returns the count."""
    import torch

    k = 0
    while k < limit:
        phase = clique.tune_info(op, nbytes)["phase"]
        if phase == "stage2" or (phase == "idle" and k >= 2):  # idle: not tunable (pinned/small)
            break
        call()
        k += 1
    torch.cuda.synchronize()
    return k


def run_config4(clique, sends, recvs, topo, args, stream) -> dict:
    """BASELINE config 4: NVLink path capped to few SMs to emulate an H800-class
    link ratio, so the balancer has real headroom to give to PCIe.

    With 8 virtual ranks on one GPU the PCIe path carries every rank's bytes
    over ONE PCIe link, i.e. 1/8 of a per-GPU link per rank.  The cap is chosen
    so NVLink-only busbw : PCIe-only busbw matches H800's 200:64 GB/s per
    direction (topo.py:130).  Then the bucket is handed to
    the in-library balancer (no flxSetShares): Stage 1 + guard on its first
    calls, Stage 2 afterwards — and timed against NVLink-only.
    """
    from paper_2510_15882_b200.links import PathKind
    from paper_2510_15882_b200.striping import CollectiveOp

    n = len(sends)
    AR = CollectiveOp.ALLREDUCE

    def busbw_pinned(shares, ctas, steps=8):
        clique.set_nvlink_ctas(ctas)
        clique.set_shares(AR, shares, AR_BYTES)
        for _ in range(2):
            clique.all_reduce(sends, recvs)
        dt = _time_steps(lambda: clique.all_reduce(sends, recvs), steps, stream)
        return busbw_allreduce(AR_BYTES, dt, n), dt

    pcie_only, _ = busbw_pinned((0, 1000, 0), 0, steps=3)
    target = pcie_only * 200.0 / 64.0
    best = None
    for ctas in (1, 2, 3, 4, 6, 8, 12, 16):
        bw, _ = busbw_pinned((1000, 0, 0), ctas, steps=3)
        if best is None or abs(bw - target) < abs(best[1] - target):
            best = (ctas, bw)
    ctas = best[0]
    nv_only, nv_dt = busbw_pinned((1000, 0, 0), ctas, steps=args.steps)
    clique.set_shares(AR, None, AR_BYTES)  # unpin: the in-library balancer owns the bucket
    t0 = time.perf_counter()
    tune_calls = settle(clique, lambda: clique.all_reduce(sends, recvs), AR, AR_BYTES)
    tune_wall = time.perf_counter() - t0
    info = clique.tune_info(AR, AR_BYTES)
    trace = clique.tune_trace(AR, AR_BYTES)
    for _ in range(2):
        clique.all_reduce(sends, recvs)
    st_dt = _time_steps(lambda: clique.all_reduce(sends, recvs), args.steps, stream)
    striped = busbw_allreduce(AR_BYTES, st_dt, n)
    pbytes = clique.path_bytes()
    exact = torch_exact(sends)
    ok = all(r.equal(exact) for r in recvs)
    drift = run_stage2_drift(clique, sends, recvs, stream)
    from paper_2510_15882_b200.calibration import CalibrationError

    try:
        cal = run_calibration(clique, sends, recvs, stream, ctas, striped, pbytes, info)
    except CalibrationError as e:  # e.g. timings distorted by a profiler: report, go on
        cal = {"error": f"calibration infeasible on this run's rows: {e}"}
    clique.set_nvlink_ctas(args.nvlink_ctas)
    return {
        "workload": "config 4: AllReduce fp32 256 MiB/rank, 8 virtual ranks, NVLink-path kernel "
                    "capped to emulate H800's NVLink:PCIe ratio (200:64 per direction)",
        "nvlink_ctas": ctas, "pcie_only_busbw": round(pcie_only, 2),
        "nvlink_only_busbw": round(nv_only, 2), "striped_busbw": round(striped, 2),
        "gain_pct": round(100 * (striped / nv_only - 1), 2),
        "shares": {k.short: info["shares"][int(k)] for k in PathKind},
        "traffic_share_pct": {k.short: round(100 * pbytes[k] / AR_BYTES, 3) for k in PathKind},
        "balancer": {"where": "in-library, no flxSetShares", "tuning_calls": tune_calls,
                     "tuning_wall_s": round(tune_wall, 2), **info,
                     "stage1_trace": [r["action"] for r in trace]},
        "ms_per_step": {"nvlink_only": round(nv_dt * 1e3, 4), "striped": round(st_dt * 1e3, 4)},
        "result_exact": bool(ok),
        "stage2_drift": drift,
        "calibration": cal,
    }


def run_calibration(clique, sends, recvs, stream, ctas, striped_busbw, pbytes, info) -> dict:
    """SURVEY §8(f) row 2 on this run's own rows: the alpha-beta fit of the
    reference's `calibrate` (bench.py:151-227, calibration.py) over NVLink-only
    AllReduce at 3 sizes under the config-4 cap plus the balancer's striped row,
    then Stage 1 re-run seeded from the calibrated topology (flxSetLinkProfile)
    instead of the in-call probe round."""
    from paper_2510_15882_b200 import calibration as C
    from paper_2510_15882_b200.links import PathKind
    from paper_2510_15882_b200.striping import CollectiveOp

    AR = CollectiveOp.ALLREDUCE
    n = len(sends)
    rows = []
    for mib in (64, 128, 256):
        cnt = mib * MIB // 4
        s = [x[:cnt] for x in sends]
        r = [x[:cnt] for x in recvs]
        clique.set_shares(AR, (1000, 0, 0), cnt * 4)
        for _ in range(2):
            clique.all_reduce(s, r)
        dt = _time_steps(lambda: clique.all_reduce(s, r), 5, stream)
        rows.append(C.MeasuredRow(AR, n, cnt * 4, C.MODE_BASELINE, cnt * 4 / dt / 1e9))
        if mib != 256:
            clique.set_shares(AR, None, cnt * 4)
    clique.set_shares(AR, None, AR_BYTES)
    algbw_striped = striped_busbw / (2 * (n - 1) / n)
    load = 100.0 * pbytes[PathKind.PCIE_STAGED] / AR_BYTES
    if load <= 0:  # the balancer kept NVLink-only: no striped row to fit PCIe from
        cal = C.calibrate(rows)
        fit = cal.nvlink[(AR, n)]
        return {"rows": [{"size": r.size, "mode": r.mode, "algbw_gbs": round(r.algbw, 3)}
                         for r in rows],
                "nvlink_fit": {"bandwidth_gbs": round(fit.bandwidth / 1e9, 3),
                               "latency_us": round(fit.latency * 1e6, 3)},
                "pcie_fit_gbs": None, "note": "no striped row (balancer kept NVLink-only)"}
    rows.append(C.MeasuredRow(AR, n, AR_BYTES, C.MODE_PCIE_ONLY, algbw_striped, 0, load))
    cal = C.calibrate(rows)
    topo = C.build_calibrated_topology(cal, AR, n, C.MODE_PCIE_ONLY)
    clique.set_link_profile(topo)  # resets the bucket: Stage 1 again, seeded from the fit
    calls = settle(clique, lambda: clique.all_reduce(sends, recvs), AR, AR_BYTES)
    seeded = clique.tune_info(AR, AR_BYTES)
    clique.set_link_profile(None)
    fit = cal.nvlink[(AR, n)]
    return {"rows": [{"size": r.size, "mode": r.mode, "algbw_gbs": round(r.algbw, 3),
                      "pcie_load_pct": round(r.pcie_load, 2)} for r in rows],
            "nvlink_fit": {"bandwidth_gbs": round(fit.bandwidth / 1e9, 3),
                           "latency_us": round(fit.latency * 1e6, 3),
                           "residuals": {str(k): round(v, 4) for k, v in fit.residuals.items()}},
            "pcie_fit_gbs": round(cal.secondary[(AR, n, C.MODE_PCIE_ONLY)][PathKind.PCIE_STAGED]
                                  / 1e9, 3),
            "stage1_seeded_from_fit": {"tuning_calls": calls,
                                       "iterations": seeded["stage1_iterations"],
                                       "shares": seeded["shares"],
                                       "tuned_ms": seeded["tuned_ms"],
                                       "kept_tuned": seeded["kept_tuned"]},
            "stage1_seeded_by_probe_round": {"iterations": info["stage1_iterations"],
                                             "shares": info["shares"]}}


def torch_exact(sends):
    import torch

    return torch.stack(list(sends)).sum(0)


def run_stage2_drift(clique, sends, recvs, stream, calls: int = 240, hog_from: int = 60,
                     hog_to: int = 150) -> dict:
    """In-library Stage 2 on the real path (balancer.py:163-207 semantics, csrc/autotune.cpp):
    in the config-4 setting, a competing H2D stream hogs PCIe between calls hog_from and
    hog_to.  The balancer sees the PCIe path slow down (lagged CUDA-event times), moves
    granules to NVLink, and moves them back once the hog stops."""
    import torch

    from paper_2510_15882_b200.links import PathKind
    from paper_2510_15882_b200.striping import CollectiveOp

    AR = CollectiveOp.ALLREDUCE
    hog_src = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
    hog_dst = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    hog_stream = torch.cuda.Stream()
    start = clique.tune_info(AR, AR_BYTES)
    seen = start["stage2_evaluations"]
    trace = []
    for call in range(1, calls + 1):
        hog = hog_from <= call < hog_to
        if hog:
            with torch.cuda.stream(hog_stream):
                hog_dst.copy_(hog_src, non_blocking=True)
        clique.all_reduce(sends, recvs)
        # lockstep: one hog copy per call, so the contention lasts exactly the
        # hog window (the host would otherwise queue them all ahead of the GPU)
        stream.synchronize()
        info = clique.tune_info(AR, AR_BYTES)
        if info["stage2_evaluations"] != seen:
            seen = info["stage2_evaluations"]
            ev = clique.tune_evaluations(AR, AR_BYTES)[-1]
            trace.append({"call": call, "gap": None if ev["gap"] is None else round(ev["gap"], 4),
                          "moved": ev["moved"], "pcie": info["shares"][int(PathKind.PCIE_STAGED)],
                          "hog": hog})
    torch.cuda.synchronize()
    end = clique.tune_info(AR, AR_BYTES)
    during = [e["pcie"] for e in trace if e["hog"]]
    return {"calls": calls, "hog_calls": [hog_from, hog_to],
            "pcie_granules_start": start["shares"][int(PathKind.PCIE_STAGED)],
            "pcie_granules_during_hog_min": min(during) if during else None,
            "pcie_granules_end": end["shares"][int(PathKind.PCIE_STAGED)],
            "evaluations": trace}


def run_config5(clique, topo, stream) -> dict:
    """BASELINE config 5: Qwen2.5-32B-shaped TP=8 prefill at 64K tokens
    (hidden 5120, intermediate 27648, 64 layers).  Each layer's
    two row-parallel GEMMs (attention out-projection [64K, 640] x [640, 5120]
    and MLP down-projection [64K, 3456] x [3456, 5120] per rank) each end in an
    AllReduce of the [65536, 5120] bf16 activation (640 MiB per rank) — here
    over 8 virtual ranks on one B200, so all 8 ranks' GEMMs share this GPU too.

    Reported: the AllReduces alone (comm), the GEMMs alone, the full layer
    stack GEMM -> AllReduce in order, and the same stack with each GEMM+AllReduce
    pair split into 4 token chunks on two streams so chunk k's AllReduce overlaps
    chunk k+1's GEMM (the comm/compute overlap a fused TP layer gets)."""
    import torch

    from paper_2510_15882_b200.links import PathKind
    from paper_2510_15882_b200.striping import CollectiveOp

    n, tokens, hidden, layers = len(clique.comms), 65536, 5120, 64
    k_attn, k_mlp = 5120 // 8, 27648 // 8
    nbytes = tokens * hidden * 2
    g = torch.Generator(device="cuda").manual_seed(55)
    outs = [torch.empty(tokens, hidden, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    x_attn = [torch.randn(tokens, k_attn, device="cuda", generator=g).bfloat16() for _ in range(n)]
    x_mlp = [torch.randn(tokens, k_mlp, device="cuda", generator=g).bfloat16() for _ in range(n)]
    w_attn = [(torch.randn(k_attn, hidden, device="cuda", generator=g) / 32).bfloat16()
              for _ in range(n)]
    w_mlp = [(torch.randn(k_mlp, hidden, device="cuda", generator=g) / 64).bfloat16()
             for _ in range(n)]
    AR = CollectiveOp.ALLREDUCE

    # comm alone: 128 AllReduces of 640 MiB (the balancer settles the bucket first)
    acts = [torch.randn(tokens, hidden, device="cuda", generator=g).bfloat16() for _ in range(n)]
    settle(clique, lambda: clique.all_reduce(acts, outs), AR, nbytes)
    comm_s = _time_steps(lambda: clique.all_reduce(acts, outs), 2 * layers, stream) * 2 * layers
    acc = acts[0].float()
    for x in acts[1:]:
        acc += x.float()
    exact = all(torch.equal(o, acc.bfloat16()) for o in outs)
    info = clique.tune_info(AR, nbytes)
    b = clique.path_bytes()
    del acts, acc

    def gemms(which, rows=None):
        xs, ws = (x_attn, w_attn) if which == 0 else (x_mlp, w_mlp)
        for r in range(n):
            if rows is None:
                torch.matmul(xs[r], ws[r], out=outs[r])
            else:
                torch.matmul(xs[r][rows], ws[r], out=outs[r][rows])

    def gemm_only():
        for _ in range(layers):
            gemms(0)
            gemms(1)

    def sequential():
        for _ in range(layers):
            for which in (0, 1):
                gemms(which)
                clique.all_reduce(outs, outs)  # in place, after the GEMM on the same stream

    chunks = 4
    per = tokens // chunks
    comm_stream = torch.cuda.Stream()
    ev_gemm = [torch.cuda.Event() for _ in range(chunks)]
    ev_comm = torch.cuda.Event()
    views = [[o[c * per:(c + 1) * per] for o in outs] for c in range(chunks)]
    settle(clique, lambda: clique.all_reduce(views[0], views[0]), AR, nbytes // chunks)

    def chunked():
        for _ in range(layers):
            for which in (0, 1):
                stream.wait_event(ev_comm)  # the previous AllReduce finished with outs
                for c in range(chunks):
                    gemms(which, slice(c * per, (c + 1) * per))
                    ev_gemm[c].record(stream)
                    comm_stream.wait_event(ev_gemm[c])
                    clique.all_reduce(views[c], views[c], stream=comm_stream)
                ev_comm.record(comm_stream)
        stream.wait_event(ev_comm)

    out = {}
    for name, fn in (("gemm_only", gemm_only), ("sequential", sequential), ("chunked", chunked)):
        fn()  # warm (cuBLAS heuristics, balancer on the chunk bucket)
        out[name] = _time_steps(fn, 1, stream)
    flops = 2.0 * tokens * hidden * (k_attn + k_mlp) * n * layers
    del x_attn, x_mlp, w_attn, w_mlp, outs, views
    torch.cuda.empty_cache()
    return {"workload": "config 5: Qwen2.5-32B TP=8 prefill, 64K tokens, 64 layers x (GEMM -> "
                        "AllReduce [65536,5120] bf16) x 2, 8 virtual ranks on one B200",
            "calls": 2 * layers, "comm_only_ms": round(comm_s * 1e3, 2),
            "per_call_ms": round(comm_s / (2 * layers) * 1e3, 4),
            "busbw": round(busbw_allreduce(nbytes, comm_s / (2 * layers), n), 2),
            "gemm_only_ms": round(out["gemm_only"] * 1e3, 2),
            "gemm_tflops": round(flops / out["gemm_only"] / 1e12, 1),
            "layers_sequential_ms": round(out["sequential"] * 1e3, 2),
            "layers_chunked_overlap_ms": round(out["chunked"] * 1e3, 2),
            "comm_share_of_sequential_pct": round(100 * comm_s / out["sequential"], 1),
            "overlap_saved_ms": round((out["sequential"] - out["chunked"]) * 1e3, 2),
            "shares": {k.short: info["shares"][int(k)] for k in PathKind},
            "traffic_share_pct": {k.short: round(100 * b[k] / nbytes, 3) for k in PathKind},
            "fixed_order_fp32_fold_exact": exact}


# --------------------------------------------------------------- N > 1
def run_multi_gpu(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2510_15882_b200 import comm as flx
    from paper_2510_15882_b200.links import PathKind
    from paper_2510_15882_b200.striping import CollectiveOp

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2510_15882_b200.probe import probe_pcie
    from paper_2510_15882_b200.striping import ShareDistribution

    c = flx.Communicator.from_process_group()
    if args.nvlink_ctas:
        c.set_nvlink_ctas(args.nvlink_ctas)
    count = AR_BYTES // 4
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    send = torch.randint(-1024, 1024, (count,), device="cuda", generator=gen).float()
    recv = torch.empty_like(send)
    stream = torch.cuda.current_stream()
    # measured PCIe of this rank's link (the north star's aggregate-link roofline
    # adds it to NVLink's 900 GB/s); min over ranks
    pc = torch.tensor([probe_pcie(64 << 20, reps=3)["h2d"] / 1e9], device="cuda")
    dist.all_reduce(pc, op=dist.ReduceOp.MIN)
    pcie_gbs = float(pc.item())

    def stage1(op, s, r):
        """The in-library balancer settles the bucket (Stage 1 + guard with
        rank-agreed timings through the shared host segment), or --shares pins it."""
        nbytes = s.numel() * s.element_size()
        if args.shares or world < 2:  # world 1 (FLX_BENCH_MULTI smoke): nothing to tune
            g = [int(x) for x in (args.shares or "1000,0,0").split(",")]
            shares = ShareDistribution({k: g[int(k)] for k in PathKind if g[int(k)] or k == 0})
            c.set_shares(op, shares, nbytes)
            return shares, None
        fn = (lambda: c.all_reduce(s, r)) if op == CollectiveOp.ALLREDUCE else \
            (lambda: c.all_gather(s, r))
        calls = settle(c, fn, op, nbytes)
        info = c.tune_info(op, nbytes)
        shares = ShareDistribution({k: info["shares"][int(k)] for k in PathKind
                                    if info["shares"][int(k)] or k == PathKind.NVLINK})
        return shares, {"tuning_calls": calls, **info,
                        "stage1_trace": [t["action"] for t in c.tune_trace(op, nbytes)]}

    shares, trace = stage1(CollectiveOp.ALLREDUCE, send, recv)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        dist.barrier()
        dt = _time_steps(fn, args.steps, stream)
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    launches0 = flx.launch_count()
    sampler = ClockSampler(local).start() if rank == 0 else None
    dt = timed(lambda: c.all_reduce(send, recv))
    clocks = sampler.stop() if sampler else None
    launches = flx.launch_count() - launches0
    pbytes = c.path_bytes()
    ref = send.clone()
    nccl_dt = timed(lambda: dist.all_reduce(ref))  # in place; values are irrelevant to timing
    exact = send.clone()
    dist.all_reduce(exact)  # integer-valued fp32: exact in any order
    ok = torch.equal(recv, exact)

    # e2e through the public API: this rank's input H2D from pinned memory,
    # in-place striped AllReduce, result D2H — every step.  Two device buffers:
    # step k's D2H (own stream) overlaps step k+1's H2D, as in the N=1 line.
    host_in = send.cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    work = [torch.empty_like(send), torch.empty_like(send)]
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    done_up = [torch.cuda.Event(), torch.cuda.Event()]
    done_ar = [torch.cuda.Event(), torch.cuda.Event()]
    done_down = [torch.cuda.Event(), torch.cuda.Event()]
    k_box = [0]

    def e2e_step():
        k = k_box[0] % 2
        k_box[0] += 1
        up.wait_event(done_down[k])            # buffer k drained by its last D2H
        with torch.cuda.stream(up):
            work[k].copy_(host_in, non_blocking=True)
            done_up[k].record(up)
        stream.wait_event(done_up[k])
        c.all_reduce(work[k], work[k])         # in place, public API
        done_ar[k].record(stream)
        down.wait_event(done_ar[k])
        with torch.cuda.stream(down):
            host_out.copy_(work[k], non_blocking=True)
            done_down[k].record(down)
        stream.wait_event(done_down[k])        # the step ends with its result on the host

    e2e_dt = timed(e2e_step)
    e2e_ok = torch.equal(host_out, exact.cpu())

    # AllGather bf16, 256 MiB gathered (config 2)
    ag_count = AG_OUT_BYTES // 2 // world
    ag_send = torch.randn(ag_count, device="cuda", generator=gen).bfloat16()
    ag_recv = torch.empty(ag_count * world, device="cuda", dtype=torch.bfloat16)
    ag_shares, _ = stage1(CollectiveOp.ALLGATHER, ag_send, ag_recv)
    ag_dt = timed(lambda: c.all_gather(ag_send, ag_recv))
    ag_bytes = c.path_bytes()
    ag_ref = torch.empty_like(ag_recv)
    ag_nccl_dt = timed(lambda: dist.all_gather_into_tensor(ag_ref, ag_send))
    ag_ok = torch.equal(ag_recv, ag_ref)
    del ag_send, ag_recv, ag_ref

    # ReduceScatter / AllToAll fp32 on the AllReduce inputs (8(f) row 4), NCCL beside
    extra = {}
    blk = count // world
    rs_out, rs_ref = torch.empty(blk, device="cuda"), torch.empty(blk, device="cuda")
    a2a_out, a2a_ref = torch.empty_like(send), torch.empty_like(send)
    for name, cop, ours, theirs in (
            ("reducescatter", CollectiveOp.REDUCESCATTER,
             lambda: c.reduce_scatter(send, rs_out),
             lambda: dist.reduce_scatter_tensor(rs_ref, send)),
            ("alltoall", CollectiveOp.ALLTOALL, lambda: c.all_to_all(send, a2a_out),
             lambda: dist.all_to_all_single(a2a_ref, send))):
        if args.shares or world < 2:
            g = [int(x) for x in (args.shares or "1000,0,0").split(",")]
            c.set_shares(cop, ShareDistribution({k: g[int(k)] for k in PathKind
                                                 if g[int(k)] or k == 0}), AR_BYTES // world)
        else:  # the library balances the bucket (one block = AR_BYTES / world per rank)
            settle(c, ours, cop, AR_BYTES // world)
        dt_c = timed(ours)
        dt_n = timed(theirs)
        same = torch.equal(rs_out, rs_ref) if cop == CollectiveOp.REDUCESCATTER else \
            torch.equal(a2a_out, a2a_ref)
        extra[name] = {"value": round(AR_BYTES / dt_c * (world - 1) / world / 1e9, 2),
                       "unit": "GB/s", "dtype": "f32", "ms_per_step": round(dt_c * 1e3, 4),
                       "nccl": round(AR_BYTES / dt_n * (world - 1) / world / 1e9, 2),
                       "matches_nccl_bitwise": bool(same)}
    del rs_out, rs_ref, a2a_out, a2a_ref
    cpu = cpu_allreduce_sample(5.0, AR_BYTES, world) if rank == 0 else None
    if rank == 0:
        value = busbw_allreduce(AR_BYTES, dt, world) * 1.0
        emit({
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(world),
            "shares": {k.short: shares.get(k) for k in PathKind},
            "traffic_share_pct": {k.short: round(100 * pbytes[k] / AR_BYTES, 3) for k in PathKind},
            "balancer": trace if trace else "fixed --shares",
            "roofline": {"bound": "link", "achieved": round(value, 2),
                         "peak": round(900.0 + pcie_gbs, 1), "unit": "GB/s",
                         "frac": round(value / (900.0 + pcie_gbs), 4), "traffic": None,
                         "kernel": "rank_allreduce_kernel (NVLink slice) + host-hub PCIe slice",
                         "note": "busbw vs the north star's aggregate-link roofline: NVLink 5 "
                                 "900 GB/s/dir + this run's measured PCIe H2D (min over ranks); "
                                 "NIC absent.  Same denominator as the N=1 line's link_roofline"},
            "cpu_baseline": cpu,
            "nccl": {"value": round(busbw_allreduce(AR_BYTES, nccl_dt, world), 2),
                     "ms_per_step": round(nccl_dt * 1e3, 4)},
            "result_matches_exact_sum": bool(ok), "gpu_launches": launches, "clocks": clocks,
            "e2e": {"value": round(busbw_allreduce(AR_BYTES, e2e_dt, world), 3), "unit": "GB/s",
                    "h2d_bytes_per_step": world * AR_BYTES, "d2h_bytes_per_step": world * AR_BYTES,
                    "ms_per_step": round(e2e_dt * 1e3, 3), "result_exact": bool(e2e_ok),
                    "note": "every rank moves its own 256 MiB in and out over its own PCIe link; "
                            "step k's D2H overlapped with step k+1's H2D"},
            "allgather": {
                "value": round(busbw_allgather(AG_OUT_BYTES, ag_dt, world), 2), "unit": "GB/s",
                "dtype": "bf16", "ms_per_step": round(ag_dt * 1e3, 4),
                "shares": {k.short: ag_shares.get(k) for k in PathKind},
                "traffic_share_pct": {k.short: round(100 * ag_bytes[k] / (AG_OUT_BYTES // world), 3)
                                      for k in PathKind},
                "nccl": round(busbw_allgather(AG_OUT_BYTES, ag_nccl_dt, world), 2),
                "matches_nccl_bitwise": bool(ag_ok),
                "link_roofline": link_roofline(busbw_allgather(AG_OUT_BYTES, ag_dt, world),
                                               pcie_gbs)},
            **extra,
            "link_roofline": link_roofline(value, pcie_gbs),
        })
    dist.barrier()
    c.destroy()
    dist.destroy_process_group()


def launch_ranks(args) -> int:
    """Run this benchmark as ``args.gpus`` ranks under torchrun (one process per
    GPU, NCCL/IPC between them).  Fails loudly when the box has fewer GPUs."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, this box "
                         f"has {have}; not running (no 1-GPU stand-in)\n")
        return 2
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    argv = [a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *argv]
    sys.stdout.flush()
    return subprocess.call(cmd, stdout=_JSON_FD if _JSON_FD is not None else None)


def main() -> None:
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["flexlink", "reference"], default="flexlink")
    p.add_argument("--nvlink-ctas", type=int, default=0,
                   help="cap the NVLink-path kernel's CTAs (config 4)")
    p.add_argument("--shares", default="", help="N>1: fixed granules nvlink,pcie,rdma")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--skip-config4", action="store_true")
    p.add_argument("--skip-config5", action="store_true")
    args = p.parse_args()
    if args.warmup < 3 and args.impl == "flexlink":
        args.warmup = 3
    route_native_stdout_to_stderr()
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: launch the N ranks ourselves (one process
        # per GPU, torchrun on 127.0.0.1) — never a silent 1-GPU run
        sys.exit(launch_ranks(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus and args.gpus > 1:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # FLX_BENCH_MULTI=1: take the one-process-per-GPU path even at WORLD_SIZE 1
    # (a smoke test of run_multi_gpu on a 1-GPU box)
    if world > 1 or os.environ.get("FLX_BENCH_MULTI") == "1":
        os.environ.setdefault("FLX_BOOT_TIMEOUT", "60")
        os.environ.setdefault("FLX_TIMEOUT_S", "60")  # a stalled peer ends the run, not 10 min
        try:
            run_multi_gpu(args)
        except Exception as e:  # report, do not hang the job
            if int(os.environ.get("RANK", "0")) == 0:
                emit({"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": world,
                      "error": f"{type(e).__name__}: {e}"})
            raise
    else:
        run_single_gpu(args)


if __name__ == "__main__":
    main()

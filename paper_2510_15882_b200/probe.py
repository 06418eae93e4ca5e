"""Link-profile probe: measure this box's paths and emit a linkstripe topology.

SURVEY §8(f) row 2: Stage 1 seeds its shares from per-path bandwidth
(`tuner.py:94-101` via `effective_bandwidths`), and the reference's presets stop
at H100/GB200 (`topo.py:129-135`).  This probe measures, on the GPU it runs on:

* PCIe: pinned H2D / D2H bandwidth alone and both directions at once (the
  shared-interface cap), and the per-copy latency (alpha) of a small copy;
* NVLink: with >= 2 visible GPUs, a peer copy (cudaMemcpyPeer via torch); on a
  single GPU the "NVLink" stand-in of a virtual-rank clique is the HBM fold,
  so its per-rank byte rate is measured with the fused kernel itself.

and returns a :class:`~paper_2510_15882_b200.links.TopologySpec` in the
reference's units (unidirectional bytes/s, seconds per step), or writes the
YAML document `load_topology` reads (`topo.py:210-239`).
"""

from __future__ import annotations

import statistics

from .links import DEFAULT_STAGING_CHUNK, LinkSpec, PathKind, TopologySpec

__all__ = ["probe_pcie", "probe_peer", "probe_virtual_nvlink", "probe_topology",
           "topology_to_yaml"]


def _events():
    import torch

    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time(fn, reps: int) -> float:
    import torch

    fn()
    torch.cuda.synchronize()
    a, b = _events()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def probe_pcie(nbytes: int = 256 << 20, reps: int = 5) -> dict:
    """Pinned-memory copy rates (bytes/s) and small-copy latency (s)."""
    import torch

    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    host2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h2d = nbytes / _time(lambda: dev.copy_(host, non_blocking=True), reps)
    d2h = nbytes / _time(lambda: host.copy_(dev, non_blocking=True), reps)
    side = torch.cuda.Stream()

    def both():
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            host2.copy_(dev2, non_blocking=True)
        dev.copy_(host, non_blocking=True)
        torch.cuda.current_stream().wait_stream(side)

    bidir = nbytes / _time(both, reps)
    small_h = torch.empty(4096, dtype=torch.uint8, pin_memory=True)
    small_d = torch.empty(4096, dtype=torch.uint8, device="cuda")
    lat = statistics.median(_time(lambda: small_d.copy_(small_h, non_blocking=True), 50)
                            for _ in range(3))
    return {"h2d": h2d, "d2h": d2h, "bidir_each": bidir, "latency": lat}


def probe_peer(nbytes: int = 256 << 20, reps: int = 5) -> dict | None:
    """Peer copy rate GPU0 -> GPU1 (bytes/s), or None with a single GPU."""
    import torch

    if torch.cuda.device_count() < 2:
        return None
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    rate = nbytes / _time(lambda: dst.copy_(src, non_blocking=True), reps)
    small_s = torch.empty(4096, dtype=torch.uint8, device="cuda:0")
    small_d = torch.empty(4096, dtype=torch.uint8, device="cuda:1")
    lat = _time(lambda: small_d.copy_(small_s, non_blocking=True), 50)
    return {"peer": rate, "latency": lat}


def probe_virtual_nvlink(nranks: int = 8, nbytes: int = 64 << 20, reps: int = 10) -> dict:
    """Per-rank message rate of the fused virtual-rank fold (the 1-GPU NVLink stand-in):
    bytes of one rank's message reduced per second, and the fixed cost of a tiny call."""
    import torch

    from .comm import Clique
    from .striping import CollectiveOp

    s = [torch.randn(nbytes // 4, device="cuda") for _ in range(nranks)]
    r = [torch.empty_like(x) for x in s]
    tiny = [torch.randn(64, device="cuda") for _ in range(nranks)]
    tiny_r = [torch.empty_like(x) for x in tiny]
    with Clique(nranks) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
        for _ in range(2):
            c.all_reduce(s, r)
        for _ in range(reps):
            c.all_reduce(s, r)
        t_big = statistics.median(h[PathKind.NVLINK] for h in c.comms[0].path_times_history(reps))
        for _ in range(reps):
            c.all_reduce(tiny, tiny_r)
        t_small = statistics.median(h[PathKind.NVLINK]
                                    for h in c.comms[0].path_times_history(reps))
    return {"rate": nbytes / t_big, "latency": t_small}


def probe_topology(nranks: int = 8, name: str = "probed", staging_chunk: int = 0,
                   include_pcie: bool = True) -> tuple[TopologySpec, dict]:
    """Measure and build the link profile (reference units).  With one GPU the
    NVLink entry is the virtual-rank fold; with two or more, the peer copy."""
    raw: dict = {}
    peer = probe_peer()
    if peer:
        raw["peer"] = peer
        nv = LinkSpec(PathKind.NVLINK, peer["peer"], base_latency=peer["latency"])
    else:
        v = probe_virtual_nvlink(nranks)
        raw["virtual_nvlink"] = v
        # per ring step the reference moves size/N per rank (collectives.py:167);
        # express the fold's per-rank rate as an equivalent per-direction link rate
        nv = LinkSpec(PathKind.NVLINK, v["rate"] * 2 * (nranks - 1) / nranks,
                      base_latency=v["latency"] / (2 * (nranks - 1)))
    links = {PathKind.NVLINK: nv}
    shared = 0.0
    if include_pcie:
        p = probe_pcie()
        raw["pcie"] = p
        chunk = staging_chunk or DEFAULT_STAGING_CHUNK
        links[PathKind.PCIE_STAGED] = LinkSpec(PathKind.PCIE_STAGED, p["bidir_each"],
                                               base_latency=p["latency"], staging_chunk=chunk)
        shared = max(p["h2d"], p["d2h"], p["bidir_each"])
    topo = TopologySpec(n_gpus=max(2, nranks), links=links, path_contention=include_pcie,
                        shared_interface_bw=shared, name=name)
    return topo, raw


def topology_to_yaml(topo: TopologySpec) -> str:
    """The `load_topology` document for ``topo`` (rates in GB/s, times in us)."""
    lines = [f"name: {topo.name}", f"n_gpus: {topo.n_gpus}",
             f"path_contention: {'true' if topo.path_contention else 'false'}"]
    if topo.shared_interface_bw:
        lines.append(f"shared_interface_bw: {topo.shared_interface_bw / 1e9:.6f} GB/s")
    lines.append("links:")
    for kind in topo.present_paths:
        link = topo.links[kind]
        parts = [f"bandwidth: {link.bandwidth_uni / 1e9:.6f} GB/s",
                 f"latency: {link.base_latency * 1e6:.6f}us"]
        if link.staging_chunk:
            parts.append(f"staging_chunk: {link.staging_chunk}")
        if link.per_chunk_overhead:
            parts.append(f"chunk_overhead: {link.per_chunk_overhead * 1e6:.6f}us")
        lines.append(f"  {kind.short}: {{{', '.join(parts)}}}")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    import json
    import sys

    topo, raw = probe_topology()
    text = topology_to_yaml(topo)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(text)
    print(text)
    print(json.dumps(raw))

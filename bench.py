#!/usr/bin/env python3
"""Benchmark of the subgraph-iteration hot path (BASELINE.json metric).

Default workload (N=1): configs[3] of BASELINE.json, the configuration the
metric is quoted on at 1/2/4/8 B200 -- C4: connected components on the
uniform-random (a=b=c=d=0.25) scale-27 graph, symmetrized (4.29 G directed
edges), predictive vertex updating on (strong predictor), 16 CSC pages.
`--config C1|C2|C3|C4` selects the other BASELINE configs; single flags
override a preset.  Every graph is the reference's own instance:
generate_rmat / assign_weights (ingest.cpp:112-152, std::mt19937_64, seed 0;
weights seed 1 in [1, 64]) -- generated on the GPU here and by the OpenMP
oracle in the reference arm, bit-identical streams (jump-ahead chunks).

A "step" is one pagestream::run() to convergence (PageRank: 20 iterations).
  value    = |E| * iterations / time-to-converge (graph GTEPS), graph resident
             in HBM, CUDA-event time on the engine stream, max over ranks;
  e2e      = the same metric through the public C-ABI call sr_run_graph (the
             pagestream::run drop-in) with the graph in pinned host memory:
             upload + run + values D2H inside the timed region;
  roofline = the dominant kernel (K1 pull / K8 PageRank) per launch, bytes per
             SURVEY §8(d) (plus the gathered-only model), vs MEASURED_PEAKS;
  cpu_baseline = the reference's own run() (oracle/_ref, compiled from the
             reference sources) on the box's host cores, same graph and config
             (PageRank: the OpenMP fp64 oracle -- the reference has none).

`--impl reference` runs the reference arm: the graph is built by the oracle
(no libseraph, no GPU) and the reference's run() is timed (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS and time-to-converge (BFS/SSSP/PR/CC, RMAT) at 1/2/4/8 B200 vs CPU ref"
ALGOS = {"bfs": 0, "cc": 1, "sssp": 2, "pagerank": 3}
MODES = {"baseline": 0, "reentry": 1, "double-buffer": 2, "pipelined": 3, "pipelined-fine": 4}
PREDS = {"off": 0, "strong": 1, "weak": 2}
RMAT = (0.57, 0.19, 0.19, 0.05)
UNIFORM = (0.25, 0.25, 0.25, 0.25)
L2_LABEL_BYTES = 126 << 20  # B200 L2 (for the workload label; the GPU arm queries the device)

# BASELINE.json configs (C5 needs 8 GPUs with host-streamed shards: not a 1-GPU preset)
PRESETS = {
    "C1": dict(algo="bfs", scale=20, uniform=False, pages=16, mode="baseline", predictor="strong",
               budget_gb=0.0),
    "C2": dict(algo="sssp", scale=24, uniform=False, pages=16, mode="pipelined",
               predictor="strong", budget_gb=0.0),
    "C3": dict(algo="pagerank", scale=26, uniform=False, pages=256, mode="baseline",
               predictor="off", budget_gb=2.0),
    "C4": dict(algo="cc", scale=27, uniform=True, pages=16, mode="baseline", predictor="strong",
               budget_gb=0.0),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4", choices=list(PRESETS))
    p.add_argument("--algo", choices=list(ALGOS))
    p.add_argument("--scale", type=int)
    p.add_argument("--edge-factor", type=int, default=16)
    p.add_argument("--uniform", action="store_true", default=None,
                   help="a=b=c=d=0.25 (uniform random)")
    p.add_argument("--rmat", dest="uniform", action="store_false",
                   help="Graph500 quadrants .57/.19/.19/.05")
    p.add_argument("--pages", type=int)
    p.add_argument("--mode", choices=list(MODES))
    p.add_argument("--predictor", choices=list(PREDS))
    p.add_argument("--window", type=int, default=8)
    p.add_argument("--mrt", type=int, default=2)
    p.add_argument("--budget-gb", type=float, help="forced HBM budget (out-of-core path)")
    p.add_argument("--pr-iters", type=int, default=20)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--exchange", default="peer", choices=["allreduce", "peer"],
                   help="N>1: peer stores into the other ranks' replicas over CUDA IPC + a "
                        "barrier per round, or the MIN all-reduce of the replicas per round")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0)
    a = p.parse_args()
    for k, v in PRESETS[a.config].items():
        if getattr(a, k) is None:
            setattr(a, k, v)
    a.weighted = a.algo == "sssp"
    a.symmetric = a.algo == "cc"
    return a


# ---------------------------------------------------------------------------
# the workload, identical in both arms
# ---------------------------------------------------------------------------
def config_name(a):
    return {"bfs": "C1", "sssp": "C5" if a.scale >= 29 else "C2", "pagerank": "C3",
            "cc": "C4"}[a.algo]


def m_est(a, n):
    """|E| of the generated graph (symmetrize doubles the RMAT edges)."""
    return n * a.edge_factor * (2 if a.symmetric else 1)


def csc_bytes(a, n, m):
    """Σ page_bytes (graph.cpp:96-100) of the page set."""
    return ((n + a.pages) + m * (2 if a.weighted else 1)) * 4


def workload_config(a, n, m):
    quad = UNIFORM if a.uniform else RMAT
    kind = "uniform" if a.uniform else "RMAT"
    label = (f"{config_name(a)}: {a.algo.upper()} {kind}-{a.scale} ef{a.edge_factor}"
             f"{' symmetrized' if a.symmetric else ''}{' w[1,64]' if a.weighted else ''}, "
             f"{a.pages} pages, {a.mode}/{a.predictor}, window {a.window}"
             f"{f', {a.pr_iters} iterations d=0.85' if a.algo == 'pagerank' else ''}"
             f"{f', HBM budget {a.budget_gb:g} GB (out-of-core)' if a.budget_gb else ''}")
    gb = csc_bytes(a, n, m)
    inst = (f"generate_rmat(scale={a.scale}, ef={a.edge_factor}, a/b/c/d={'/'.join(map(str, quad))}, "
            f"seed={a.seed}) [std::mt19937_64, ingest.cpp:112-141]")
    if a.weighted:
        inst += f" + assign_weights(seed={a.seed + 1}, 1, 64)"
    if a.symmetric:
        inst += " + symmetrize"
    cfg = {"workload": label, "algo": a.algo, "graph": kind.lower(), "quadrants": list(quad),
           "scale": a.scale, "edge_factor": a.edge_factor, "vertices": n, "edges": m,
           "pages": a.pages, "schedule": a.mode, "predictor": a.predictor, "window": a.window,
           "hbm_budget_gb": a.budget_gb or None, "instance": inst,
           "l2": ("inputs larger than L2 (CSC %.2f GB vs 126 MB L2)" % (gb / 1e9))
           if gb >= 4 * L2_LABEL_BYTES else
           ("CSC %.3f GB < 4x L2: the GPU arm flushes L2 before every step" % (gb / 1e9)),
           "parallelism": f"dp{a.gpus}" if a.gpus > 1 else "single"}
    if a.algo in ("bfs", "sssp"):
        cfg["source"] = 0
    if a.algo == "pagerank":
        cfg["iterations"] = a.pr_iters
        cfg["damping"] = 0.85
    return cfg


def degree_hash(out_off):
    """Instance fingerprint: the CSR degree sequence hashed (wrapping u64)."""
    off = np.asarray(out_off, np.uint64)
    k = np.arange(off.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) | np.uint64(1)
    with np.errstate(over="ignore"):
        return "%016x" % int(np.bitwise_xor.reduce(off * k) ^ np.uint64(off.size))


def value_signature(algo, vals):
    """Run fingerprint shared by both arms (values are bit-exact across them)."""
    v = np.asarray(vals)
    if algo == 1:
        return {"components": int(np.count_nonzero(v == np.arange(v.size, dtype=np.uint32))),
                "label_sum": int(v.astype(np.uint64).sum())}
    reach = v != 0xFFFFFFFF
    return {"reached": int(reach.sum()), "value_sum": int(v[reach].astype(np.uint64).sum())}


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i - 5] for r in rows for i in range(5, 9) if r[i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def gather_roofline(gathers_per_s, info, clocks):
    """Second bound of the pull kernels: a random 4-byte gather touches its own
    128 B line, and the L1TEX unit retires ~1 line (wavefront) per SM clock
    (B300_MICROARCH.md: rt_L1tex_wf ~ 1.0 cyc/wf), so gathers/s <= SMs x f_SM."""
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = info["sm_count"] * mhz * 1e6
    return {"achieved_gathers_per_s": round(gathers_per_s / 1e9, 2), "unit": "G/s",
            "peak": round(peak / 1e9, 2), "frac": round(gathers_per_s / peak, 4),
            "peak_basis": f"{info['sm_count']} SMs x {mhz:.0f} MHz x 1 L1TEX wavefront/cycle"}


def profile_traffic(key):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    e = d.get(key)
    return e.get("dram_bytes_per_launch") if e else None


def k1_roofline(a, runs, info, clocks, step_s):
    """K1 (dense pull, incl. source-blocked launches) per launch against HBM.
    SURVEY §8(d) per-unit bytes -- per edge 4 B in_sources (+4 B weight for
    SSSP) + 4 B gathered value, per destination 8 B (in_offsets + value; +1 B
    status under the weak predictor), per valid update 4 B -- applied to the
    units K1 actually processes: the edges it streams in (`edges_streamed`),
    the source values it gathers (`gathers`) and the destinations its phase A
    scans (`dest_visits`: once per launch, i.e. once per source block).  Edges of
    destinations that provably cannot improve (at the floor) are counted in the
    reference's edges_read but never loaded; `reference_units_model` charges
    §8(d) on edges_read as well (it exceeds 1 when such skips dominate)."""
    from paper_1806_00762_b200 import pagestream as ps
    per_src = 8 if a.weighted else 4
    per_dest = 9 if a.predictor == "weak" else 8
    b8d = bref = k1_s = 0.0
    launches = gathers = edges = streamed = 0
    for r in runs:
        for st in r.metrics.per_pass:
            if st.kind != ps.PassKind.SPARSE_PUSH:
                bref += (per_src + 4) * st.edges_read + per_dest * st.attempts + 4 * st.valid_updates
                b8d += 4 * st.valid_updates
                edges += st.edges_read
        b8d += (per_src * r.metrics.edges_streamed + 4 * r.metrics.gathers +
                per_dest * r.metrics.dest_visits)
        gathers += r.metrics.gathers
        streamed += r.metrics.edges_streamed
        k1_s += r.metrics.relax_seconds
        launches += r.metrics.relax_launches
    if not launches or k1_s <= 0:
        return None
    peak, src = measured_peaks()
    ach = b8d / k1_s / 1e9
    ref = bref / k1_s / 1e9
    return {"bound": "hbm", "kernel": "pull_relax_kernel (K1), every launch inside the timed runs",
            "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
            "peak_source": src, "traffic": profile_traffic(f"{a.algo}-s{a.scale}"),
            "model": f"SURVEY §8(d) per-unit bytes on the units K1 processes: {per_src} B/edge "
                     f"streamed + 4 B/gathered source + {per_dest} B/destination scanned + "
                     "4 B/valid update",
            "algorithmic_bytes_per_launch": int(b8d / launches),
            "launch_ms": round(k1_s / launches * 1e3, 4), "launches": launches,
            "share_of_step": round(k1_s / (step_s * len(runs)), 3),
            "units_per_run": {"edges_read_reference": edges // len(runs),
                              "edges_streamed": streamed // len(runs),
                              "gathers": gathers // len(runs),
                              "dest_visits": sum(r.metrics.dest_visits for r in runs) // len(runs)},
            "reference_units_model": {
                "achieved": round(ref, 1), "frac": round(ref / peak, 4),
                "bytes_per_launch": int(bref / launches),
                "per_unit": f"{per_src + 4} B/edge read (the reference's edges_read, incl. edges "
                            f"never loaded) + {per_dest} B/attempted destination + 4 B/valid"},
            "gather_roofline": gather_roofline(gathers / k1_s, info, clocks)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(a, rank, world, local_rank):
    from paper_1806_00762_b200 import _native as N
    from paper_1806_00762_b200 import pagestream as ps

    algo = ALGOS[a.algo]
    pr = algo == 3
    prog = ps.VertexProgram(ps.AlgoKind(algo), 0)
    cfg = ps.EngineConfig(predictor=ps.PredictorMode(PREDS[a.predictor]),
                          window_capacity=a.window, clock=ps.ClockMode.WALL,
                          pr_iterations=a.pr_iters, profile_kernels=True)
    cfg.schedule.kind = ps.ScheduleModeKind(MODES[a.mode])
    cfg.schedule.max_reentry_times = a.mrt
    budget = int(a.budget_gb * 2**30)
    quad = UNIFORM if a.uniform else RMAT
    n = 1 << a.scale
    cap = (n + a.pages - 1) // a.pages

    def sync():
        N.check(N.lib.sr_device_sync(local_rank))

    dist = torch = None
    if world > 1:
        import torch
        import torch.distributed as dist

    def world_uid():
        uid = [None]
        if rank == 0:
            buf = (N.C.c_uint8 * 128)()
            N.check(N.lib.sr_nccl_unique_id(N.C.byref(buf)))
            uid[0] = bytes(buf)
        dist.broadcast_object_list(uid, src=0)
        return uid[0]

    need_cpu = rank == 0 and world == 1 and not a.no_cpu_baseline
    need_host = (not a.no_e2e) or need_cpu
    # the push adjacency: traversals derive it on the device from the resident
    # pages; PageRank never reads it (out-degrees only)
    csr_edges = False
    t0 = time.time()
    gen = dict(seed=a.seed, weights=(1, 64, a.seed + 1) if a.weighted else None,
               symmetrize=a.symmetric, page_vertex_capacity=cap)
    arena = N.PinnedArena()
    host = None
    footprint = None
    e2e_skip = None
    if world == 1 and budget:
        # out of core: the graph is built in a scratch context and exported to
        # pinned host memory; the budgeted engine loads it from there, so its
        # device footprint (cudaMemGetInfo delta) is the budget's honest test:
        # pages + push adjacency <= budget, plus O(|V|) vertex state
        with ps.Engine(local_rank) as scratch:
            scratch.generate_graph(a.scale, a.edge_factor, *quad, csr_edges=not pr, **gen)
            host = scratch.export_graph(arena, csr_edges=not pr)
        build_s = time.time() - t0
        free0 = ps.device_info(local_rank)["free_mem"]
        eng = ps.Engine(local_rank, budget)
        eng.load_csr(host[0], with_edges=not pr)
        eng.load_pages(host[1])
        footprint = {"free_before": free0}
    elif world == 1:
        eng = ps.Engine(local_rank, budget)
        eng.generate_graph(a.scale, a.edge_factor, *quad, csr_edges=csr_edges, **gen)
        build_s = time.time() - t0
        if need_host:  # the reference's run() also needs the push adjacency
            host = eng.export_graph(arena, csr_edges=need_cpu and not pr)
    else:
        eng = ps.Engine(local_rank, budget)
        eng.attach_world(rank, world, world_uid())
        eng.set_exchange(a.exchange == "peer")
        # a sharded rank keeps only its shard: every rank generates the whole
        # graph on its own GPU (seconds) and load_pages keeps the pages of its
        # destination range and the CSR rows of its vertices (O(|E|/N))
        if not a.no_e2e:
            # the e2e leg needs the graph in host memory on every rank: only
            # when world copies fit comfortably in this node's RAM
            import psutil
            need = (n + 1) * 8 + m_est(a, n) * 4 * (2 if a.weighted else 1) * (1 if pr else 2)
            if world * need < 0.6 * psutil.virtual_memory().available:
                with ps.Engine(local_rank) as scratch:
                    scratch.generate_graph(a.scale, a.edge_factor, *quad, csr_edges=not pr,
                                           **gen)
                    host = scratch.export_graph(arena, csr_edges=not pr)
            else:
                e2e_skip = (f"{world} host copies of the graph ({world * need / 2**30:.0f} GiB) "
                            f"exceed 60 % of this node's available RAM")
        eng.generate_graph(a.scale, a.edge_factor, *quad, csr_edges=not pr, **gen)
        build_s = time.time() - t0
    m = eng.graph_info()["num_edges"]

    info = ps.device_info(local_rank)
    gbytes = csc_bytes(a, n, m)
    flush = gbytes < 4 * info["l2_bytes"]  # small inputs: evict L2 before every step

    def one(want=False):
        if flush:
            eng.flush_l2(4 * info["l2_bytes"])
        return eng.run(prog, cfg, want_values=want)

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.4)  # nvidia-smi needs a moment before its first sample
    for _ in range(max(a.warmup, 0)):
        one()
    if world > 1:
        dist.barrier()
    sync()
    dev_s, runs = [], []
    t1 = time.time()
    for _ in range(a.steps):
        r = one()
        dev_s.append(r.metrics.device_seconds)
        runs.append(r)
    sync()
    wall = time.time() - t1
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_s = sum(dev_s) / len(dev_s)
    if world > 1:
        t = torch.tensor([step_s], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_s = float(t.item())
    last = runs[-1].metrics
    iters = a.pr_iters if pr else 1
    value = m * iters / step_s / 1e9
    launches = sum(r.metrics.kernel_launches for r in runs)

    if footprint is not None:
        # vertex state: values/next/snapshot, flags, frontier lists, stamps,
        # out-degrees, u64 out-offsets and prefixes, PageRank vectors
        vs = n * (4 * 3 + 3 + 4 * 4 + 4 + 8 * 2 + (4 * 5 if pr else 0))
        used = footprint["free_before"] - ps.device_info(local_rank)["free_mem"]
        gi = eng.graph_info()
        footprint = {"device_bytes": int(used), "budget_bytes": budget,
                     "vertex_state_bytes_est": int(vs),
                     "within_budget_plus_vertex_state": bool(used <= budget + vs),
                     "adjacency_on_host": bool(gi.get("adjacency_on_host", 0)),
                     "page_bytes": int(csc_bytes(a, n, m)),
                     "adjacency_bytes": 0 if pr else int(m * (8 if a.weighted else 4)),
                     "how": "cudaMemGetInfo before the budgeted context vs after the timed runs"}

    # parity at full size: device fixpoint law + the run's value signature
    res = one(want=True)
    parity = {}
    if not pr:
        viol = eng.verify_fixpoint(ps.AlgoKind(algo), res.values)
        if world > 1:  # a sharded rank checks its own CSR rows: sum over ranks
            t = torch.tensor([viol], dtype=torch.int64, device=f"cuda:{local_rank}")
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            viol = int(t.item())
        parity["fixpoint_violations"] = viol
        parity["signature"] = value_signature(algo, res.values)
        if algo != 1:
            parity["source_value"] = int(res.values[0])

    # roofline of the dominant kernel
    roof = None
    if a.budget_gb:
        # out-of-core: the host link bounds; streamed bytes per run / run time
        gbps = N.C.c_double()
        N.check(N.lib.sr_bench_h2d(local_rank, 1 << 30, 3, N.C.byref(gbps)))
        streamed = last.bytes_transferred
        ach = streamed / step_s / 1e9
        kern = "pr_pull_kernel (K8)" if pr else "pull_relax_kernel (K1) + push (K3)"
        roof = {"bound": "host-link", "kernel": kern + " + H2D page stream",
                "achieved": round(ach, 2), "peak": round(gbps.value, 2), "unit": "GB/s",
                "frac": round(ach / gbps.value, 4),
                "peak_source": "measured (sr_bench_h2d, pinned 1 GiB, this run)",
                "traffic": None, "streamed_bytes_per_run": int(streamed),
                "model": "page_bytes of every admitted page (graph.cpp:96-100)"}
    elif pr:
        alg = (8 * m + 16 * n) * iters
        k8_s = sum(r.metrics.relax_seconds for r in runs) / len(runs)
        k8_l = sum(r.metrics.relax_launches for r in runs) / len(runs)
        peak, src = measured_peaks()
        ach = alg / k8_s / 1e9
        roof = {"bound": "hbm", "kernel": "pr_pull_kernel (K8), every launch of the timed runs",
                "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "peak_source": src,
                "traffic": profile_traffic(f"pagerank-s{a.scale}"),
                "model": "SURVEY §8(d): 8 B/edge + 16 B/destination per iteration",
                "algorithmic_bytes_per_launch": int(alg / max(k8_l, 1)),
                "launch_ms": round(k8_s / max(k8_l, 1) * 1e3, 4), "launches": int(k8_l),
                "share_of_step": round(k8_s / step_s, 3),
                "gather_roofline": gather_roofline(m * iters / k8_s, info, clocks)}
    else:
        roof = k1_roofline(a, runs, info, clocks, step_s)
        if roof:
            ms, edges = eng.bench_pull_sweep(ps.AlgoKind(algo), 10)
            roof["isolated_sweep"] = {"ms": round(ms, 4), "edges": edges,
                                      "note": "gate-off K1 sweep over the converged values"}

    # the multi-pass subgraph-iteration schedules on the same resident graph
    schedules = {}
    if not pr and world == 1 and not a.budget_gb:
        for mode in ("baseline", "reentry", "pipelined"):
            if mode == a.mode:
                continue
            c2 = ps.EngineConfig(predictor=cfg.predictor, window_capacity=a.window,
                                 clock=ps.ClockMode.WALL)
            c2.schedule.kind = ps.ScheduleModeKind(MODES[mode])
            eng.run(prog, c2, want_values=False)
            t = min(eng.run(prog, c2, want_values=False).metrics.device_seconds for _ in range(3))
            schedules[mode] = {"ms": round(t * 1e3, 3), "gteps": round(m * iters / t / 1e9, 2)}

    # e2e: the public C-ABI one-shot call with pinned host buffers
    e2e = None
    if e2e_skip:
        e2e = {"value": None, "unit": "GTEPS", "skipped": e2e_skip}
    elif not a.no_e2e:
        # the CSR offsets only: the engine derives the push adjacency from the
        # pages -- unless a budget keeps pages + adjacency from fitting: then the
        # adjacency is passed and stays in pinned host memory (zero-copy pushes)
        if (budget or world > 1) and not pr and host[0].out_neighbors.size:
            csr = host[0]  # sharded ranks upload only their own rows of it
        else:
            csr = ps.CsrGraph(n, host[0].out_offsets, np.zeros(0, np.uint32),
                              np.zeros(0, np.uint32))
        pages = host[1]
        e2e_eng = ps.Engine(local_rank, budget)
        if world > 1:
            e2e_eng.attach_world(rank, world, world_uid())
            e2e_eng.set_exchange(a.exchange == "peer")
        vals = arena.array(n, np.float32 if pr else np.uint32)  # reused output (values / ranks)
        e2e_eng.run_graph(csr, pages, prog, cfg, values_out=vals)  # warm-up
        sync()
        if world > 1:
            dist.barrier()
        reps = max(1, min(a.steps, 5))
        t2 = time.time()
        for _ in range(reps):
            rr = e2e_eng.run_graph(csr, pages, prog, cfg, values_out=vals)
        sync()
        e2e_s = (time.time() - t2) / reps
        h2d = int(csr.out_offsets.nbytes + sum(p.in_offsets.nbytes + p.in_sources.nbytes +
                                               p.in_weights.nbytes for p in pages.pages))
        d2h = n * 4
        up = rr.metrics.upload_seconds
        if world > 1:
            tt = torch.tensor([e2e_s, float(h2d), float(d2h), up], dtype=torch.float64,
                              device=f"cuda:{local_rank}")
            mx = tt.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            e2e_s, h2d, d2h, up = float(mx[0]), int(tt[1]), int(tt[2]), float(mx[3])
        e2e = {"value": round(m * iters / e2e_s / 1e9, 4), "unit": "GTEPS",
               "seconds_per_step": round(e2e_s, 5), "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "upload_seconds": round(up, 5),
               "h2d_bytes_measured": int(rr.metrics.h2d_bytes),
               "call": "sr_run_graph (pagestream::run drop-in), pinned host inputs"
                       + (", one shard per GPU, max over ranks" if world > 1 else "")}
        if world == 1:
            # the C++ drop-in's callers pass std::vector (pageable) arrays: same
            # call from pageable copies (the engine stages them through pinned
            # chunks on several host threads, csrc/stager.cpp)
            csr_p = ps.CsrGraph(n, np.array(csr.out_offsets), csr.out_neighbors,
                                csr.out_weights)
            pages_p = ps.PageSet(pages.num_vertices, pages.page_vertex_capacity, pages.weighted,
                                 [ps.CscPage(p.vertex_begin, p.vertex_end, np.array(p.in_offsets),
                                             np.array(p.in_sources), np.array(p.in_weights))
                                  for p in pages.pages])
            vals_p = np.zeros(n, np.float32 if pr else np.uint32)  # reused, pages touched
            e2e_eng.run_graph(csr_p, pages_p, prog, cfg, values_out=vals_p)  # warm-up
            sync()
            t3 = time.time()
            for _ in range(reps):
                rp = e2e_eng.run_graph(csr_p, pages_p, prog, cfg, values_out=vals_p)
            sync()
            pg_s = (time.time() - t3) / reps
            e2e["pageable"] = {"value": round(m * iters / pg_s / 1e9, 4),
                               "seconds_per_step": round(pg_s, 5),
                               "upload_seconds": round(rp.metrics.upload_seconds, 5),
                               "call": "sr_run_graph from pageable host arrays (what the C++ "
                                       "drop-in pagestream::seraph::run passes)"}
            del csr_p, pages_p
        e2e_eng.close()

    # CPU baseline on this box's host cores (rank 0, N=1), same graph
    cpu = None
    instance = {"degree_hash": degree_hash(host[0].out_offsets)} if host else {}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a, host, n, m, res)
        for k in ("bit_exact_vs_reference_run", "pagerank"):
            if k in cpu:
                parity[k] = cpu.pop(k)

    ms_per_step = step_s * 1e3
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32" if pr else "u32", "data": "synthetic",
        "config": workload_config(a, n, m),
        "time_to_converge_ms": round(ms_per_step, 4),
        "gteps_read": round(last.edges_read / dev_s[-1] / 1e9, 4),
        "passes": {"total": last.passes, "dense": last.dense_passes, "sparse": last.sparse_passes,
                   "recovery": last.recovery_passes, "edges_read": last.edges_read},
        "wall_ms_per_step": round(wall / a.steps * 1e3, 4),
        "e2e": e2e, "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu,
        **({"device_footprint": footprint} if footprint else {}),
        "clocks": clocks, "parity": parity, "schedules": schedules,
        "instance": instance,
        "build": {"graph_build_s": round(build_s, 2),
                  "how": "device: sr_generate_graph (mt19937_64 jump-ahead chunks) + stable "
                         "radix-sort build_csr/build_csc_pages",
                  "l2_flush_per_step": bool(flush)},
    }
    if world > 1:
        out["config"]["exchange"] = a.exchange
    eng.close()
    arena.close()
    if rank == 0:
        print(json.dumps(out), flush=True)


def cpu_baseline(a, host, n, m, res):
    """The reference's run() (oracle/_ref) on this box's host cores, same graph and
    config, one full run (bounded sample); reports whether its values are
    bit-identical to ours.  PageRank: the OpenMP fp64 oracle (the reference has
    none) -- timed as the baseline and used as the checker of our ranks."""
    from oracle import oracle as O
    cores = a.cpu_threads or os.cpu_count() or 1
    csr, pages, in_off, in_src, in_w = host
    algo = ALGOS[a.algo]
    if algo == 3:
        t = time.time()
        want = O.pagerank_par(n, in_off, in_src, csr.out_offsets, a.pr_iters, 0.85, cores)
        t = time.time() - t
        mx, mr, l1 = O.pr_compare(res.ranks, want, 1e-12, cores)
        return {"value": round(m * a.pr_iters / t / 1e9, 5), "unit": "GTEPS", "cores": cores,
                "kind": "port", "seconds": round(t, 3),
                "sample": f"1 full fp64 PageRank ({a.pr_iters} iterations) by the OpenMP "
                          "oracle (oracle_pagerank_par) on the same graph",
                "pagerank": {"max_abs": mx, "max_rel": mr, "l1_sum": l1,
                             "rel_floor": 1e-12, "checker": "oracle_pagerank_par (fp64)"}}
    ref = O.load_reference()
    if ref is None:
        return None
    # the push adjacency exported from the device (derived from the pages: the
    # order within a source may differ from build_csr's, which run()'s values
    # do not depend on)
    g = O.RefGraph(ref, n, csr.out_offsets, csr.out_neighbors,
                   csr.out_weights if a.weighted else None, in_off, in_src,
                   in_w if a.weighted else None, (n + a.pages - 1) // a.pages)
    vals, mets = g.run(algo, 0, PREDS[a.predictor], MODES[a.mode], a.mrt, 3, a.window, cores,
                       1, 0, 0.05, want_values=True)
    g.close()
    t = mets["wall_seconds"]
    return {"bit_exact_vs_reference_run": bool(np.array_equal(vals, res.values)),
            "value": round(m / t / 1e9, 5), "unit": "GTEPS", "cores": cores, "kind": "reference",
            "seconds": round(t, 3),
            "sample": f"1 full reference run() of the same workload (ClockMode::Wall, "
                      f"{cores} OpenMP workers)",
            "edges_read": mets["edges_read"], "passes": mets["passes"]}


# ---------------------------------------------------------------------------
# reference arm: oracle-built graph (no libseraph, no GPU), the reference's run()
# ---------------------------------------------------------------------------
def ref_workload(a, cores):
    from oracle import oracle as O
    quad = UNIFORM if a.uniform else RMAT
    n = 1 << a.scale
    src, dst = O.generate_rmat_par(a.scale, a.edge_factor, *quad, seed=a.seed, threads=cores)
    w = O.assign_weights_par(src.size, a.seed + 1, 1, 64, cores) if a.weighted else None
    if a.symmetric:
        src, dst, w = O.symmetrize_par(src, dst, w, cores)
    out_off, out_nbr, out_w = O.build_adjacency_par(n, src, dst, w, cores)
    in_off, in_src, in_w = O.build_adjacency_par(n, dst, src, w, cores)
    return n, int(src.size), (out_off, out_nbr, out_w, in_off, in_src, in_w)


def run_reference(a, rank):
    if rank != 0:
        return
    from oracle import oracle as O
    cores = a.cpu_threads or os.cpu_count() or 1
    algo = ALGOS[a.algo]
    t0 = time.time()
    n, m, (out_off, out_nbr, out_w, in_off, in_src, in_w) = ref_workload(a, cores)
    build_s = time.time() - t0
    iters = a.pr_iters if algo == 3 else 1
    ref = O.load_reference()
    if algo == 3:
        kind, what = "port", ("the OpenMP fp64 PageRank oracle (oracle_pagerank_par): the "
                              "reference has no PageRank (SPEC.md:8)")
        del out_nbr, out_w

        def one(want=False):
            t = time.time()
            r = O.pagerank_par(n, in_off, in_src, out_off, a.pr_iters, 0.85, cores)
            return time.time() - t, None, r
    else:
        if ref is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        kind, what = "reference", "the reference's run() (oracle/_ref, ClockMode::Wall)"
        g = O.RefGraph(ref, n, out_off, out_nbr, out_w, in_off, in_src, in_w,
                       (n + a.pages - 1) // a.pages)
        del out_nbr, out_w, in_src, in_w

        def one(want=False):
            vals, met = g.run(algo, 0, PREDS[a.predictor], MODES[a.mode], a.mrt, 3, a.window,
                              cores, 1, 0, 0.05, want_values=want)
            return met["wall_seconds"], met, vals

    # the reference's CPU run() has nothing to warm beyond first-touch page
    # faults: at most one untimed run keeps the arm within a few minutes
    warm = min(max(a.warmup, 0), 1)
    for _ in range(warm):
        one()
    secs, met, vals = [], None, None
    for i in range(a.steps):
        s, met, vals = one(want=i == a.steps - 1)
        secs.append(s)
    t = sum(secs) / len(secs)
    value = m * iters / t / 1e9
    parity = {}
    if algo != 3 and vals is not None:
        parity["signature"] = value_signature(algo, vals)
        if algo != 1:
            parity["source_value"] = int(vals[0])
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "GTEPS",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "warmup_runs_done": warm,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if algo == 3 else "u32", "data": "synthetic",
        "config": workload_config(a, n, m),
        "cpu_baseline": {"value": round(value, 5), "unit": "GTEPS", "cores": cores, "kind": kind,
                         "sample": f"one full run per step: {what}, {cores} threads"},
        "e2e": {"value": round(value, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "parity": parity, "instance": {"degree_hash": degree_hash(out_off)},
        "build": {"graph_build_s": round(build_s, 2),
                  "how": "oracle (OpenMP): generate_rmat/assign_weights jump-ahead chunks, "
                         "symmetrize, stable counting-sort build_csr/build_csc"},
    }
    if met is not None:
        out["passes"] = met["passes"]
        out["edges_read"] = met["edges_read"]
    if algo != 3:
        g.close()
    print(json.dumps(out), flush=True)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    a.gpus = max(a.gpus, world)
    if a.impl == "reference":
        run_reference(a, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    run_ours(a, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

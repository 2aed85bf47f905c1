"""Python mirror of the reference's public API for the hot path.

Names, fields and argument meaning follow proj/include/pagestream/*.hpp so a
caller of ``pagestream::run(csr, pages, program, config)`` (engine.hpp:125)
finds the same vocabulary here: EdgeList / CsrGraph / CscPage / PageSet
(graph.hpp), VertexProgram + make_bfs/make_cc/make_sssp (programs.hpp),
EngineConfig / ScheduleMode / TransferModel (engine.hpp, scheduler.hpp),
PassStats / MetricsReport (metrics.hpp), RunResult, and the exception classes
of errors.hpp.  The work is done by libseraph.so on the GPU; graph building
uses the library's parallel host builders.  PageRank is an addition
(AlgoKind.PAGERANK) that the reference does not have.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from ._native import (ConfigError, ContractError, DataError, Error, FormatError,  # noqa: F401
                      InputError, ParseError)

kUnreached = N.UNREACHED  # types.hpp:14
kEntryBytes = 4           # types.hpp:18


class AlgoKind(enum.IntEnum):  # types.hpp:20 (+ PAGERANK)
    BFS = N.ALGO_BFS
    CC = N.ALGO_CC
    SSSP = N.ALGO_SSSP
    PAGERANK = N.ALGO_PAGERANK


class PredictorMode(enum.IntEnum):  # predictor.hpp:12
    OFF = N.PRED_OFF
    STRONG = N.PRED_STRONG
    WEAK = N.PRED_WEAK


class ScheduleModeKind(enum.IntEnum):  # scheduler.hpp:31-37
    BASELINE = N.SCHED_BASELINE
    REENTRY = N.SCHED_REENTRY
    DOUBLE_BUFFER = N.SCHED_DOUBLE_BUFFER
    PIPELINED = N.SCHED_PIPELINED
    PIPELINED_FINE = N.SCHED_PIPELINED_FINE


_MODE_NAMES = {"baseline": ScheduleModeKind.BASELINE, "reentry": ScheduleModeKind.REENTRY,
               "double-buffer": ScheduleModeKind.DOUBLE_BUFFER,
               "pipelined": ScheduleModeKind.PIPELINED,
               "pipelined-fine": ScheduleModeKind.PIPELINED_FINE}


def parse_schedule_mode(name: str) -> ScheduleModeKind:  # scheduler.cpp:28-35
    if name not in _MODE_NAMES:
        raise ConfigError(f"unknown scheduler mode '{name}'")
    return _MODE_NAMES[name]


def parse_predictor(name: str) -> PredictorMode:  # bench.cpp:72-77
    table = {"off": PredictorMode.OFF, "strong": PredictorMode.STRONG, "weak": PredictorMode.WEAK}
    if name not in table:
        raise ConfigError(f"unknown predictor mode '{name}'")
    return table[name]


def parse_algo(name: str) -> AlgoKind:  # bench.cpp:65-70
    table = {"bfs": AlgoKind.BFS, "cc": AlgoKind.CC, "sssp": AlgoKind.SSSP,
             "pagerank": AlgoKind.PAGERANK}
    if name not in table:
        raise ConfigError(f"unknown algorithm '{name}'")
    return table[name]


class ClockMode(enum.IntEnum):  # engine.hpp:15
    VIRTUAL = N.CLOCK_VIRTUAL
    WALL = N.CLOCK_WALL


class ExecutionPolicy(enum.IntEnum):  # engine.hpp:16
    DENSITY_SWITCHED = N.EXEC_DENSITY_SWITCHED
    FORCE_SPARSE = N.EXEC_FORCE_SPARSE
    FORCE_DENSE = N.EXEC_FORCE_DENSE


class PassKind(enum.IntEnum):  # metrics.hpp:12
    SPARSE_PUSH = 0
    DENSE_PULL = 1
    RECOVERY = 2


class TraceEventKind(enum.IntEnum):  # scheduler.hpp:55
    XFER_START = 0
    XFER_END = 1
    KERNEL_START = 2
    KERNEL_END = 3
    REENTRY = 4


# ---------------------------------------------------------------------------
# Graph structures (graph.hpp)
# ---------------------------------------------------------------------------
def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


@dataclass
class EdgeList:
    """graph.hpp:19-27.  Edges as parallel src/dst arrays; weights empty when unweighted."""
    num_vertices: int = 0
    src: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    dst: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    weights: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    @staticmethod
    def from_pairs(n: int, edges, weights=None) -> "EdgeList":
        e = np.asarray(list(edges), dtype=np.uint64).reshape(-1, 2)
        w = np.zeros(0, np.uint32) if weights is None or len(weights) == 0 else _u32(weights)
        return EdgeList(int(n), _u32(e[:, 0]), _u32(e[:, 1]), w)

    def weighted(self) -> bool:
        return self.weights.size > 0

    def num_edges(self) -> int:
        return int(self.src.size)

    def validate(self) -> None:  # graph.cpp:9-22
        if self.weighted() and self.weights.size != self.src.size:
            raise InputError(f"edge list: weight array length {self.weights.size} does not match "
                             f"edge count {self.src.size}")
        if self.src.size:
            bad = np.nonzero((self.src >= self.num_vertices) | (self.dst >= self.num_vertices))[0]
            if bad.size:
                i = int(bad[0])
                raise InputError(f"edge {i} ({self.src[i]},{self.dst[i]}) has id >= num_vertices "
                                 f"{self.num_vertices}")
        if self.weighted() and self.weights.size and int(self.weights.min()) < 1:
            i = int(np.argmin(self.weights))
            raise InputError(f"edge {i} has weight < 1")


@dataclass
class CsrGraph:
    """graph.hpp:30-41."""
    num_vertices: int
    out_offsets: np.ndarray   # u64 [|V|+1]
    out_neighbors: np.ndarray  # u32 [|E|]
    out_weights: np.ndarray    # u32 [|E|] or empty

    def weighted(self) -> bool:
        return self.out_weights.size > 0

    def num_edges(self) -> int:
        # from the offsets: a lean CsrGraph (offsets only) has no adjacency arrays
        return int(self.out_offsets[-1]) if self.out_offsets.size else int(self.out_neighbors.size)

    def lean(self) -> bool:
        """Offsets only: the engine derives the push adjacency from the resident pages."""
        return self.out_neighbors.size == 0 and self.num_edges() > 0

    def out_degree(self, u: int) -> int:
        return int(self.out_offsets[u + 1] - self.out_offsets[u])


@dataclass
class CscPage:
    """graph.hpp:46-55: destination range [vertex_begin, vertex_end) with
    page-local u32 in_offsets, in_sources and optional in_weights."""
    vertex_begin: int
    vertex_end: int
    in_offsets: np.ndarray
    in_sources: np.ndarray
    in_weights: np.ndarray

    def range(self) -> int:
        return self.vertex_end - self.vertex_begin

    def edge_count(self) -> int:
        return int(self.in_sources.size)


@dataclass
class PageSet:
    """graph.hpp:57-65."""
    num_vertices: int
    page_vertex_capacity: int
    weighted: bool
    pages: List[CscPage]

    def num_edges(self) -> int:
        return sum(p.edge_count() for p in self.pages)

    def page_count(self) -> int:
        return len(self.pages)


def build_csr(el: EdgeList, threads: int = 0) -> CsrGraph:
    """Counting sort by source, input order kept within a source (graph.cpp:30-48)."""
    el.validate()
    n, m = el.num_vertices, el.num_edges()
    off = np.zeros(n + 1, np.uint64)
    nbr = np.empty(m, np.uint32)
    w = np.empty(m if el.weighted() else 0, np.uint32)
    if n:
        N.check(N.lib.sr_build_csr(n, m, N.ptr(el.src), N.ptr(el.dst), N.ptr(el.weights),
                                   N.ptr(off), N.ptr(nbr), N.ptr(w), threads))
    return CsrGraph(n, off, nbr, w)


def build_csc_pages(el: EdgeList, page_vertex_capacity: int, threads: int = 0) -> PageSet:
    """Cut the CSC into ceil(|V|/cap) pages with page-local u32 offsets (graph.cpp:50-94).
    Pages are views into three contiguous arrays (local offsets, sources, weights)."""
    if page_vertex_capacity < 1:
        raise ConfigError("page_vertex_capacity must be >= 1")
    el.validate()
    n, m, cap = el.num_vertices, el.num_edges(), int(page_vertex_capacity)
    off = np.zeros(n + 1, np.uint64)
    srcs = np.empty(m, np.uint32)
    w = np.empty(m if el.weighted() else 0, np.uint32)
    if n:
        N.check(N.lib.sr_build_csc(n, m, N.ptr(el.src), N.ptr(el.dst), N.ptr(el.weights),
                                   N.ptr(off), N.ptr(srcs), N.ptr(w), threads))
    return pages_from_csc(n, cap, off, srcs, w)


def pages_from_csc(n: int, cap: int, in_offsets_global: np.ndarray, in_sources: np.ndarray,
                   in_weights: np.ndarray, local_offsets: Optional[np.ndarray] = None) -> PageSet:
    """PageSet view over a global CSC (in_offsets u64 [|V|+1])."""
    npg = (n + cap - 1) // cap
    if local_offsets is None:
        local_offsets = np.empty(n + npg, np.uint32)
        if n:
            N.check(N.lib.sr_page_offsets(n, cap, N.ptr(in_offsets_global), N.ptr(local_offsets)))
    weighted = in_weights.size > 0
    pages = []
    for p in range(npg):
        vb, ve = p * cap, min((p + 1) * cap, n)
        lo, hi = int(in_offsets_global[vb]), int(in_offsets_global[ve])
        pages.append(CscPage(vb, ve, local_offsets[vb + p: ve + p + 1], in_sources[lo:hi],
                             in_weights[lo:hi] if weighted else np.zeros(0, np.uint32)))
    return PageSet(n, cap, weighted, pages)


def page_bytes(page: CscPage, weighted: bool, entry_bytes: int = kEntryBytes) -> int:
    """graph.cpp:96-100."""
    entries = page.in_offsets.size + page.in_sources.size
    if weighted:
        entries += page.in_sources.size
    return int(entries) * entry_bytes


def symmetrize(el: EdgeList, threads: int = 0) -> EdgeList:
    """Append the reverse of every edge, interleaved as in graph.cpp:102-118."""
    el.validate()
    m = el.num_edges()
    src = np.empty(2 * m, np.uint32)
    dst = np.empty(2 * m, np.uint32)
    w = np.empty(2 * m if el.weighted() else 0, np.uint32)
    if m:
        N.check(N.lib.sr_symmetrize(m, N.ptr(el.src), N.ptr(el.dst), N.ptr(el.weights),
                                    N.ptr(src), N.ptr(dst), N.ptr(w), threads))
    return EdgeList(el.num_vertices, src, dst, w)


def resolve_page_capacity(configured: int, num_vertices: int) -> int:
    """engine.cpp:51-54: default 32 pages."""
    if configured > 0:
        return configured
    return max(1, (num_vertices + 31) // 32)


def generate_rmat_fast(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, d=0.05,
                       seed: int = 0, threads: int = 0) -> EdgeList:
    """generate_rmat (ingest.cpp:112-141) bit-for-bit on all host threads: the
    reference's single std::mt19937_64 stream cut into chunks by GF(2)
    jump-ahead (csrc/mt64.h)."""
    n = 1 << scale
    m = n * edge_factor
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    N.check(N.lib.sr_rmat_generate(scale, edge_factor, a, b, c, d, seed, N.ptr(src), N.ptr(dst),
                                   threads))
    return EdgeList(n, src, dst, np.zeros(0, np.uint32))


def generate_rmat_device(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, d=0.05,
                         seed: int = 0, weights=None, device: int = 0) -> EdgeList:
    """generate_rmat (+ assign_weights when weights=(lo, hi, seed)) on the GPU --
    the reference's std::mt19937_64 streams, one warp per jump-ahead chunk --
    copied back: bit-identical to the reference and the host generator."""
    n = 1 << scale
    m = n * edge_factor
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    w = np.empty(m if weights else 0, np.uint32)
    lo, hi, ws = weights if weights else (0, 0, 0)
    N.check(N.lib.sr_rmat_generate_device(device, scale, edge_factor, a, b, c, d, seed, N.ptr(src),
                                          N.ptr(dst), ws, lo, hi, N.ptr(w)))
    return EdgeList(n, src, dst, w)


def assign_weights_fast(el: EdgeList, seed: int, lo: int, hi: int, threads: int = 0) -> EdgeList:
    if lo < 1:
        raise ConfigError("minimum weight must be >= 1 (non-positive weights break SSSP)")
    if lo > hi:
        raise ConfigError("weight range is empty: lo > hi")
    w = np.empty(el.num_edges(), np.uint32)
    N.check(N.lib.sr_weights_generate(el.num_edges(), seed, lo, hi, N.ptr(w), threads))
    return EdgeList(el.num_vertices, el.src, el.dst, w)


def shard_plan(num_vertices: int, in_offsets_global: np.ndarray, parts: int) -> np.ndarray:
    """Edge-balanced contiguous destination cut used by the multi-GPU path."""
    cuts = np.zeros(parts + 1, np.uint32)
    N.check(N.lib.sr_shard_plan(num_vertices, N.ptr(np.ascontiguousarray(in_offsets_global,
                                                                         dtype=np.uint64)),
                                parts, N.ptr(cuts)))
    return cuts


# ---------------------------------------------------------------------------
# Vertex programs (programs.hpp)
# ---------------------------------------------------------------------------
@dataclass
class VertexProgram:
    kind: AlgoKind = AlgoKind.BFS
    source: int = 0

    def uses_weights(self) -> bool:
        return self.kind == AlgoKind.SSSP


def make_bfs(source: int, num_vertices: int) -> VertexProgram:  # programs.cpp:9-14
    if source >= num_vertices:
        raise ConfigError(f"bfs source {source} out of range [0, {num_vertices})")
    return VertexProgram(AlgoKind.BFS, source)


def make_cc() -> VertexProgram:
    return VertexProgram(AlgoKind.CC, 0)


def make_sssp(source: int, num_vertices: int, graph_weighted: bool) -> VertexProgram:
    if source >= num_vertices:
        raise ConfigError(f"sssp source {source} out of range [0, {num_vertices})")
    if not graph_weighted:
        raise ConfigError("sssp requires a weighted graph")
    return VertexProgram(AlgoKind.SSSP, source)


def make_pagerank() -> VertexProgram:
    return VertexProgram(AlgoKind.PAGERANK, 0)


# ---------------------------------------------------------------------------
# Configuration (engine.hpp:39-52, scheduler.hpp:19-47)
# ---------------------------------------------------------------------------
@dataclass
class TransferModel:
    bytes_per_time_unit: float = 11.0
    edges_per_time_unit_per_worker: float = 1.75
    worker_count: int = 4


@dataclass
class ScheduleMode:
    kind: ScheduleModeKind = ScheduleModeKind.BASELINE
    max_reentry_times: int = 2
    buffer_repetitions: int = 3


@dataclass
class EngineConfig:
    page_vertex_capacity: int = 0
    density_threshold_fraction: float = 0.05
    predictor: PredictorMode = PredictorMode.OFF
    schedule: ScheduleMode = field(default_factory=ScheduleMode)
    window_capacity: int = 8
    transfer: TransferModel = field(default_factory=TransferModel)
    clock: ClockMode = ClockMode.VIRTUAL
    execution: ExecutionPolicy = ExecutionPolicy.DENSITY_SWITCHED
    seed: int = 0
    record_trace: bool = False
    # PageRank (new)
    pr_iterations: int = 20
    pr_damping: float = 0.85
    profile_kernels: bool = False  # time K1/K8 launches (MetricsReport.relax_seconds)

    def validate(self) -> None:  # engine.cpp:43-49
        if self.window_capacity < 2:
            raise ConfigError("window capacity must be >= 2")
        if not (0.0 < self.density_threshold_fraction <= 1.0):
            raise ConfigError("density threshold fraction must be in (0, 1]")
        if self.transfer.bytes_per_time_unit <= 0 or self.transfer.edges_per_time_unit_per_worker <= 0:
            raise ConfigError("transfer model rates must be positive")
        if self.transfer.worker_count < 1:
            raise ConfigError("worker_count must be >= 1")
        if self.schedule.kind == ScheduleModeKind.REENTRY and self.schedule.max_reentry_times < 1:
            raise ConfigError("max reentry times must be >= 1")
        if self.schedule.kind == ScheduleModeKind.DOUBLE_BUFFER and self.schedule.buffer_repetitions < 1:
            raise ConfigError("double-buffer repetitions must be >= 1")

    def to_c(self, program: VertexProgram) -> N.RunConfig:
        c = N.default_config()
        c.algo = int(program.kind)
        c.source = int(program.source)
        c.predictor = int(self.predictor)
        c.schedule = int(self.schedule.kind)
        c.max_reentry_times = int(self.schedule.max_reentry_times)
        c.buffer_repetitions = int(self.schedule.buffer_repetitions)
        c.window_capacity = int(self.window_capacity)
        c.density_threshold_fraction = float(self.density_threshold_fraction)
        c.bytes_per_time_unit = float(self.transfer.bytes_per_time_unit)
        c.edges_per_time_unit_per_worker = float(self.transfer.edges_per_time_unit_per_worker)
        c.worker_count = int(self.transfer.worker_count)
        c.clock = int(self.clock)
        c.execution = int(self.execution)
        c.record_trace = 1 if self.record_trace else 0
        c.seed = int(self.seed)
        c.pr_iterations = int(self.pr_iterations)
        c.pr_damping = float(self.pr_damping)
        c.profile_kernels = 1 if self.profile_kernels else 0
        return c


# ---------------------------------------------------------------------------
# Results (metrics.hpp, engine.hpp:117-121)
# ---------------------------------------------------------------------------
@dataclass
class PassStats:
    pass_index: int = 0
    kind: PassKind = PassKind.SPARSE_PUSH
    attempts: int = 0
    valid_updates: int = 0
    skipped: int = 0
    edges_read: int = 0
    changed_vertices: int = 0
    status_counts: List[int] = field(default_factory=lambda: [0] * 6)
    has_status_counts: bool = False


@dataclass
class MetricsReport:
    passes: int = 0
    sparse_passes: int = 0
    dense_passes: int = 0
    recovery_passes: int = 0
    pages_transferred: int = 0
    bytes_transferred: int = 0
    update_attempts: int = 0
    valid_updates: int = 0
    skipped_vertices: int = 0
    edges_read: int = 0
    virtual_makespan: float = 0.0
    wall_seconds: float = 0.0
    per_pass: List[PassStats] = field(default_factory=list)
    prediction_accuracy: Optional[float] = None
    # B200 extras
    device_seconds: float = 0.0
    upload_seconds: float = 0.0
    kernel_launches: int = 0
    kernel_runs: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    relax_seconds: float = 0.0
    relax_launches: int = 0
    gathers: int = 0
    edges_streamed: int = 0
    dest_visits: int = 0

    def throughput(self) -> float:  # metrics.hpp:51-56
        t = self.wall_seconds if self.wall_seconds > 0 else self.virtual_makespan
        return self.edges_read / t if t > 0 else 0.0


@dataclass
class TraceEvent:
    time: float
    kind: TraceEventKind
    page_id: int
    pass_index: int


@dataclass
class RunResult:
    values: np.ndarray                 # u32 per vertex (BFS/CC/SSSP)
    metrics: MetricsReport
    trace: List[TraceEvent] = field(default_factory=list)
    ranks: Optional[np.ndarray] = None  # f32 per vertex (PageRank)


_TRACE_NAMES = {TraceEventKind.XFER_START: "xfer_start", TraceEventKind.XFER_END: "xfer_end",
                TraceEventKind.KERNEL_START: "kernel_start", TraceEventKind.KERNEL_END: "kernel_end",
                TraceEventKind.REENTRY: "reentry"}


def write_trace_csv(trace) -> str:  # scheduler.cpp:60-67
    """Virtual clock: model time units; Wall clock: milliseconds of CUDA events."""
    out = ["event_time,event_kind,page_id,pass_index"]
    for e in trace:
        out.append(f"{e.time:.6f},{_TRACE_NAMES[TraceEventKind(e.kind)]},{e.page_id},{e.pass_index}")
    return "\n".join(out) + "\n"


def simulate_pass_makespan(pass_trace) -> float:  # scheduler.cpp:69-77
    if not pass_trace:
        return 0.0
    ts = [e.time for e in pass_trace]
    return max(ts) - min(ts)


def write_status_histogram_csv(report: MetricsReport) -> str:  # metrics.cpp:9-27
    rows = [p for p in report.per_pass if p.has_status_counts]
    if not rows:
        raise DataError("no status histograms recorded; run with the weak predictor")
    out = ["pass,s0,s1,s2,s3,s4,s5,attempted,skipped,real"]
    for i, p in enumerate(rows):
        s = p.status_counts
        out.append(",".join(str(x) for x in [i, *s, s[0] + s[1] + s[5], s[2] + s[3] + s[4],
                                              p.changed_vertices]))
    return "\n".join(out) + "\n"


def _metrics_from_c(m: N.MetricsC, passes) -> MetricsReport:
    r = MetricsReport()
    for f in ("passes", "sparse_passes", "dense_passes", "recovery_passes", "pages_transferred",
              "bytes_transferred", "update_attempts", "valid_updates", "skipped_vertices",
              "edges_read", "virtual_makespan", "wall_seconds", "device_seconds",
              "upload_seconds", "kernel_launches", "kernel_runs", "h2d_bytes", "d2h_bytes",
              "relax_seconds", "relax_launches", "gathers", "edges_streamed",
              "dest_visits"):
        setattr(r, f, getattr(m, f))
    if m.has_prediction_accuracy:
        r.prediction_accuracy = m.prediction_accuracy
    for p in passes:
        r.per_pass.append(PassStats(p.pass_index, PassKind(p.kind), p.attempts, p.valid_updates,
                                    p.skipped, p.edges_read, p.changed_vertices,
                                    list(p.status_counts), bool(p.has_status_counts)))
    return r


# ---------------------------------------------------------------------------
# Engine (one libseraph context on one device)
# ---------------------------------------------------------------------------
def _page_views(pages: PageSet):
    arr = (N.PageView * max(1, len(pages.pages)))()
    for i, p in enumerate(pages.pages):
        for a in (p.in_offsets, p.in_sources, p.in_weights):
            assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
        arr[i].vertex_begin = p.vertex_begin
        arr[i].vertex_end = p.vertex_end
        arr[i].in_offsets = N.ptr(p.in_offsets)
        arr[i].in_sources = N.ptr(p.in_sources)
        arr[i].in_weights = N.ptr(p.in_weights) if pages.weighted else None
        arr[i].edge_count = p.in_sources.size
    return arr


class Engine:
    """A libseraph context: load a graph once, run many programs on it."""

    def __init__(self, device: int = 0, hbm_budget_bytes: int = 0):
        h = C.c_void_p()
        N.check(N.lib.sr_open(device, int(hbm_budget_bytes), C.byref(h)))
        self._h = h
        self.device = device
        self.num_vertices = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib.sr_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- upload ----
    def load(self, csr: CsrGraph, pages: PageSet) -> None:
        self.load_csr(csr)
        self.load_pages(pages)

    def load_csr(self, csr: CsrGraph, with_edges: bool = True) -> None:
        # |E| from the offsets: a lean CsrGraph (offsets only) has no adjacency
        m = int(csr.out_offsets[-1]) if csr.out_offsets.size else 0
        if with_edges and csr.out_neighbors.size != m:
            raise InputError("csr: out_neighbors length does not match out_offsets[-1]")
        N.check(N.lib.sr_load_csr(self._h, csr.num_vertices, m,
                                  N.ptr(csr.out_offsets),
                                  N.ptr(csr.out_neighbors) if with_edges else None,
                                  N.ptr(csr.out_weights) if with_edges else None), self._h)
        self.num_vertices = csr.num_vertices

    def load_pages(self, pages: PageSet) -> None:
        views = _page_views(pages)
        N.check(N.lib.sr_load_pages(self._h, pages.num_vertices, pages.page_vertex_capacity,
                                    1 if pages.weighted else 0, views, len(pages.pages)), self._h)

    # ---- device-side graph build ----
    def build_graph(self, el: EdgeList, page_vertex_capacity: int, csr_edges: bool = True) -> None:
        """build_csr + build_csc_pages (graph.cpp:30-94) on the GPU from a host
        edge list; the result is resident as if loaded with load()/load_pages()."""
        if page_vertex_capacity < 1:
            raise ConfigError("page_vertex_capacity must be >= 1")
        if el.weighted() and el.weights.size and int(el.weights.min()) < 1:
            raise InputError("edge weight < 1")
        N.check(N.lib.sr_build_graph(self._h, el.num_vertices, el.num_edges(), N.ptr(el.src),
                                     N.ptr(el.dst), N.ptr(el.weights) if el.weighted() else None,
                                     int(page_vertex_capacity),
                                     N.BUILD_CSR_EDGES if csr_edges else 0), self._h)
        self.num_vertices = el.num_vertices

    def generate_graph(self, scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, d=0.05,
                       seed: int = 0, weights=None, symmetrize: bool = False,
                       page_vertex_capacity: int = 0, csr_edges: bool = True) -> None:
        """generate_rmat_fast (+ assign_weights_fast(seed=weights[2], lo, hi) when
        weights=(lo, hi, seed), + symmetrize) and the build, all on the device."""
        n = 1 << scale
        spec = N.GraphSpec(scale, edge_factor, a, b, c, d, seed, 0, 0, 0, 1 if symmetrize else 0,
                           page_vertex_capacity or (n + 15) // 16)
        if weights is not None:
            spec.weight_lo, spec.weight_hi, spec.weight_seed = weights
        N.check(N.lib.sr_generate_graph(self._h, C.byref(spec),
                                        N.BUILD_CSR_EDGES if csr_edges else 0), self._h)
        self.num_vertices = n

    def load_srph(self, path: str, page_vertex_capacity: int, csr_edges: bool = True) -> None:
        """load_binary (ingest.cpp:176-218) + build + load, on the device."""
        N.check(N.lib.sr_load_srph(self._h, os.fsencode(path), int(page_vertex_capacity),
                                   N.BUILD_CSR_EDGES if csr_edges else 0), self._h)
        self.num_vertices = self.graph_info()["num_vertices"]

    def graph_info(self) -> dict:
        gi = N.GraphInfo()
        N.check(N.lib.sr_graph_info_get(self._h, C.byref(gi)), self._h)
        return {k: getattr(gi, k) for k, _ in N.GraphInfo._fields_ if k != "pad_"}

    def export_graph(self, arena=None, csr_edges: bool = True):
        """(CsrGraph, PageSet, in_offsets, in_sources, in_weights): copies of the loaded
        graph in the reference layouts (global CSC arrays behind the page views; arrays
        from `arena.array` when given, e.g. pinned host memory)."""
        gi = self.graph_info()
        n, m = gi["num_vertices"], gi["num_edges"]
        mk = (lambda k, dt: arena.array(k, dt)) if arena is not None else (lambda k, dt: np.empty(k, dt))
        out_off = mk(n + 1, np.uint64)
        want_nbr = csr_edges and gi["has_csr_edges"]
        nbr = mk(m if want_nbr else 0, np.uint32)
        ow = mk(m if (want_nbr and gi["csr_weighted"]) else 0, np.uint32)
        in_off = np.empty(n + 1, np.uint64)
        srcs = mk(m, np.uint32)
        iw = mk(m if gi["weighted"] else 0, np.uint32)
        N.check(N.lib.sr_export_graph(self._h, N.ptr(out_off), N.ptr(nbr) if want_nbr else None,
                                      N.ptr(ow) if ow.size else None, N.ptr(in_off), N.ptr(srcs),
                                      N.ptr(iw) if iw.size else None), self._h)
        cap = gi["page_vertex_capacity"]
        npg = (n + cap - 1) // cap
        local = mk(n + npg, np.uint32)
        if n:
            N.check(N.lib.sr_page_offsets(n, cap, N.ptr(in_off), N.ptr(local)))
        return (CsrGraph(n, out_off, nbr, ow),
                pages_from_csc(n, cap, in_off, srcs, iw, local), in_off, srcs, iw)

    def attach_loopback(self, rank: int, world: int, group: str, peer: bool = False) -> None:
        """Test/dev: rank of an in-process world whose exchange goes through host
        memory (sr_attach_loopback); drive each rank's run() from its own thread.
        peer=True: improvements go straight into the other ranks' replicas."""
        N.check(N.lib.sr_attach_loopback(self._h, rank, world, group.encode(), 1 if peer else 0),
                self._h)

    def attach_world(self, rank: int, world: int, unique_id: bytes) -> None:
        uid = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        N.check(N.lib.sr_attach_world(self._h, rank, world, C.byref(uid)), self._h)

    def set_exchange(self, peer: bool) -> None:
        """Exchange of the attached world: False = MIN all-reduce of the value
        replicas per round (default); True = peer stores into the other ranks'
        replicas + a barrier (NCCL worlds: replicas mapped over CUDA IPC)."""
        N.check(N.lib.sr_set_exchange(self._h, 1 if peer else 0), self._h)

    # ---- run ----
    def run(self, program: VertexProgram, config: EngineConfig, values_out=None,
            want_values: bool = True) -> RunResult:
        config.validate()
        cfg = config.to_c(program)
        n = self.num_vertices
        vals = None
        ranks = None
        if program.kind == AlgoKind.PAGERANK:  # values_out: an f32 array for the ranks
            ranks = values_out if values_out is not None else (np.empty(n, np.float32)
                                                                if want_values else None)
        else:
            vals = values_out if values_out is not None else (np.empty(n, np.uint32)
                                                              if want_values else None)
        m = N.MetricsC()
        cap = 4096
        passes = (N.PassStatsC * cap)()
        npass = C.c_uint32()
        N.check(N.lib.sr_run(self._h, C.byref(cfg), N.ptr(vals), N.ptr(ranks), C.byref(m),
                             passes, cap, C.byref(npass)), self._h)
        res = RunResult(vals if vals is not None else np.zeros(0, np.uint32),
                        _metrics_from_c(m, passes[:min(npass.value, cap)]), ranks=ranks)
        if config.record_trace:
            res.trace = self.trace()
        return res

    def run_graph(self, csr: CsrGraph, pages: PageSet, program: VertexProgram,
                  config: EngineConfig, values_out=None) -> RunResult:
        """One call = pagestream::run(csr, pages, program, config): upload, run, download."""
        config.validate()
        _check_structures(csr, pages, program)
        cfg = config.to_c(program)
        n = csr.num_vertices
        vals = ranks = None
        if program.kind == AlgoKind.PAGERANK:  # values_out: an f32 array for the ranks
            ranks = values_out if values_out is not None else np.empty(n, np.float32)
        else:
            vals = values_out if values_out is not None else np.empty(n, np.uint32)
        views = _page_views(pages)
        m = N.MetricsC()
        cap = 4096
        passes = (N.PassStatsC * cap)()
        npass = C.c_uint32()
        N.check(N.lib.sr_run_graph(self._h, n, csr.num_edges(), N.ptr(csr.out_offsets),
                                   N.ptr(csr.out_neighbors), N.ptr(csr.out_weights),
                                   pages.page_vertex_capacity, 1 if pages.weighted else 0,
                                   views, len(pages.pages),
                                   C.byref(cfg), N.ptr(vals), N.ptr(ranks), C.byref(m), passes,
                                   cap, C.byref(npass)), self._h)
        self.num_vertices = n
        res = RunResult(vals if vals is not None else np.zeros(0, np.uint32),
                        _metrics_from_c(m, passes[:min(npass.value, cap)]), ranks=ranks)
        if config.record_trace:
            res.trace = self.trace()
        return res

    def flush_l2(self, nbytes: int = 512 << 20) -> None:
        N.check(N.lib.sr_flush_l2(self._h, int(nbytes)), self._h)

    def trace(self) -> List[TraceEvent]:
        n = C.c_uint64()
        N.check(N.lib.sr_get_trace(self._h, None, 0, C.byref(n)), self._h)
        buf = (N.TraceEventC * max(1, n.value))()
        N.check(N.lib.sr_get_trace(self._h, buf, n.value, C.byref(n)), self._h)
        return [TraceEvent(e.time, TraceEventKind(e.kind), e.page_id, e.pass_index)
                for e in buf[:n.value]]

    def verify_fixpoint(self, kind: AlgoKind, values: Optional[np.ndarray] = None) -> int:
        v = C.c_uint64()
        N.check(N.lib.sr_verify_fixpoint(self._h, int(kind),
                                         N.ptr(_u32(values)) if values is not None else None,
                                         C.byref(v)), self._h)
        return v.value

    def bench_pull_sweep(self, kind: AlgoKind, reps: int):
        ms = C.c_double()
        e = C.c_uint64()
        N.check(N.lib.sr_bench_pull_sweep(self._h, int(kind), reps, C.byref(ms), C.byref(e)),
                self._h)
        return ms.value, e.value


def _check_structures(csr: CsrGraph, pages: PageSet, program: VertexProgram) -> None:
    # engine.cpp:423-431
    if csr.num_vertices != pages.num_vertices:
        raise ConfigError("csr and page set disagree on vertex count")
    if program.uses_weights() and (not (csr.weighted() or csr.lean()) or not pages.weighted):
        raise ConfigError("sssp requires weighted graph structures")
    if program.kind in (AlgoKind.BFS, AlgoKind.SSSP) and program.source >= csr.num_vertices:
        raise ConfigError("source vertex out of range")


class Group:
    """A multi-GPU world inside this process (sr_group_*): rank r on
    devices[r], one host thread per rank inside every call; distinct devices
    talk NCCL (+ peer stores with exchange="peer"), a repeated device uses the
    in-process loopback transport.  Each rank holds its destination shard of
    the pages and its own CSR rows only."""

    def __init__(self, devices, hbm_budget_bytes: int = 0, exchange: str = "allreduce"):
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        flags = N.EXCHANGE_PEER if exchange == "peer" else 0
        N.check(N.lib.sr_group_open(arr, len(devices), int(hbm_budget_bytes), flags, C.byref(h)))
        self._h = h
        self.devices = list(devices)
        self.num_vertices = 0

    def close(self) -> None:
        if self._h:
            N.lib.sr_group_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self) -> int:
        return N.lib.sr_group_size(self._h)

    def graph_info(self, rank: int = 0) -> dict:
        gi = N.GraphInfo()
        N.check(N.lib.sr_group_graph_info(self._h, rank, C.byref(gi)), group=self._h)
        return {k: getattr(gi, k) for k, _ in N.GraphInfo._fields_}

    def load_graph(self, csr: CsrGraph, pages: PageSet, algo_hint: int = -1) -> None:
        views = _page_views(pages)
        N.check(N.lib.sr_group_load_graph(self._h, csr.num_vertices, csr.num_edges(),
                                          N.ptr(csr.out_offsets), N.ptr(csr.out_neighbors),
                                          N.ptr(csr.out_weights), pages.page_vertex_capacity,
                                          1 if pages.weighted else 0, views, len(pages.pages),
                                          int(algo_hint)), group=self._h)
        self.num_vertices = csr.num_vertices

    def _result(self, fn, program, config, n):
        cfg = config.to_c(program)
        vals = ranks = None
        if program.kind == AlgoKind.PAGERANK:
            ranks = np.empty(n, np.float32)
        else:
            vals = np.empty(n, np.uint32)
        m = N.MetricsC()
        cap = 4096
        passes = (N.PassStatsC * cap)()
        npass = C.c_uint32()
        N.check(fn(cfg, vals, ranks, m, passes, cap, npass), group=self._h)
        return RunResult(vals if vals is not None else np.zeros(0, np.uint32),
                         _metrics_from_c(m, passes[:min(npass.value, cap)]), ranks=ranks)

    def run(self, program: VertexProgram, config: EngineConfig) -> RunResult:
        config.validate()
        return self._result(lambda cfg, v, r, m, p, cap, np_: N.lib.sr_group_run(
            self._h, C.byref(cfg), N.ptr(v), N.ptr(r), C.byref(m), p, cap, C.byref(np_)),
            program, config, self.num_vertices)

    def run_graph(self, csr: CsrGraph, pages: PageSet, program: VertexProgram,
                  config: EngineConfig) -> RunResult:
        """pagestream::run over the group: every rank uploads its shard, runs, rank 0's values."""
        config.validate()
        _check_structures(csr, pages, program)
        views = _page_views(pages)
        self.num_vertices = csr.num_vertices
        return self._result(lambda cfg, v, r, m, p, cap, np_: N.lib.sr_group_run_graph(
            self._h, csr.num_vertices, csr.num_edges(), N.ptr(csr.out_offsets),
            N.ptr(csr.out_neighbors), N.ptr(csr.out_weights), pages.page_vertex_capacity,
            1 if pages.weighted else 0, views, len(pages.pages), C.byref(cfg), N.ptr(v),
            N.ptr(r), C.byref(m), p, cap, C.byref(np_)), program, config, csr.num_vertices)


_default_engines: dict = {}
_default_lock = threading.Lock()


def run(csr: CsrGraph, pages: PageSet, program: VertexProgram, config: EngineConfig,
        device: int = 0, hbm_budget_bytes: int = 0, devices=None) -> RunResult:
    """pagestream::run (engine.hpp:125-126) on the GPU; `devices` (or the
    SERAPH_DEVICES environment variable, e.g. "0,1,2,3") shards it over
    several GPUs of this process (Group)."""
    if devices is None and os.environ.get("SERAPH_DEVICES"):
        devices = [int(x) for x in os.environ["SERAPH_DEVICES"].split(",") if x.strip()]
    with _default_lock:
        # ClockMode::Virtual (the reference's deterministic schedule) runs on
        # the first device alone, as in the C++ drop-in
        if devices is not None and len(devices) > 1 and config.clock == ClockMode.WALL:
            key = ("group", tuple(devices), int(hbm_budget_bytes))
            grp = _default_engines.get(key)
            if grp is None:
                grp = Group(devices, hbm_budget_bytes)
                _default_engines[key] = grp
            return grp.run_graph(csr, pages, program, config)
        if devices:
            device = devices[0]
        key = (device, int(hbm_budget_bytes))
        eng = _default_engines.get(key)
        if eng is None:
            eng = Engine(device, hbm_budget_bytes)
            _default_engines[key] = eng
        return eng.run_graph(csr, pages, program, config)


def device_info(device: int = 0) -> dict:
    d = N.DeviceInfo()
    N.check(N.lib.sr_device_query(device, C.byref(d)))
    return {"name": d.name.decode(), "sm_count": d.sm_count, "l2_bytes": d.l2_bytes,
            "cc": f"{d.cc_major}.{d.cc_minor}", "total_mem": d.total_mem, "free_mem": d.free_mem}

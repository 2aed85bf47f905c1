"""ctypes binding of libseraph.so (include/seraph.h).

The shared library is the product: every compute call goes through it.  There
is no Python or CPU fallback -- if the library is missing this module raises
at import time, and every failing C call raises the exception class that the
reference would throw (proj/include/pagestream/errors.hpp:8-28).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SERAPH_LIB") or os.path.join(_HERE, "libseraph.so")


class Error(RuntimeError):
    """pagestream::Error (errors.hpp:8)."""


class InputError(Error):
    """Malformed graph data (errors.hpp:13)."""


class ConfigError(Error):
    """Invalid configuration (errors.hpp:16)."""


class ParseError(Error):
    """Text parsing failure (errors.hpp:19)."""


class FormatError(Error):
    """Binary graph file violates the format (errors.hpp:22)."""


class ContractError(Error):
    """Broken internal contract (errors.hpp:25)."""


class DataError(Error):
    """Report requested without its data (errors.hpp:28)."""


class CudaError(Error):
    """Device failure (maps to pagestream::Error)."""


SR_OK = 0
_CODES = {
    -1: ConfigError,
    -2: InputError,
    -3: ContractError,
    -4: DataError,
    -5: FormatError,
    -6: ParseError,
    -7: CudaError,
    -8: Error,
    -9: CudaError,
    -10: Error,
}

# enums (seraph.h)
ALGO_BFS, ALGO_CC, ALGO_SSSP, ALGO_PAGERANK = 0, 1, 2, 3
PRED_OFF, PRED_STRONG, PRED_WEAK = 0, 1, 2
SCHED_BASELINE, SCHED_REENTRY, SCHED_DOUBLE_BUFFER, SCHED_PIPELINED, SCHED_PIPELINED_FINE = range(5)
CLOCK_VIRTUAL, CLOCK_WALL = 0, 1
EXEC_DENSITY_SWITCHED, EXEC_FORCE_SPARSE, EXEC_FORCE_DENSE = 0, 1, 2
UNREACHED = 0xFFFFFFFF


class PageView(C.Structure):
    _fields_ = [
        ("vertex_begin", C.c_uint32),
        ("vertex_end", C.c_uint32),
        ("in_offsets", C.c_void_p),
        ("in_sources", C.c_void_p),
        ("in_weights", C.c_void_p),
        ("edge_count", C.c_uint64),
    ]


class RunConfig(C.Structure):
    _fields_ = [
        ("algo", C.c_int32),
        ("source", C.c_uint32),
        ("predictor", C.c_int32),
        ("schedule", C.c_int32),
        ("max_reentry_times", C.c_int32),
        ("buffer_repetitions", C.c_int32),
        ("window_capacity", C.c_uint32),
        ("density_threshold_fraction", C.c_double),
        ("bytes_per_time_unit", C.c_double),
        ("edges_per_time_unit_per_worker", C.c_double),
        ("worker_count", C.c_int32),
        ("clock", C.c_int32),
        ("execution", C.c_int32),
        ("record_trace", C.c_int32),
        ("seed", C.c_uint64),
        ("pr_iterations", C.c_uint32),
        ("pr_damping", C.c_double),
        ("profile_kernels", C.c_int32),
        ("pad_", C.c_int32),
    ]


class PassStatsC(C.Structure):
    _fields_ = [
        ("pass_index", C.c_uint32),
        ("kind", C.c_int32),
        ("attempts", C.c_uint64),
        ("valid_updates", C.c_uint64),
        ("skipped", C.c_uint64),
        ("edges_read", C.c_uint64),
        ("changed_vertices", C.c_uint64),
        ("status_counts", C.c_uint64 * 6),
        ("has_status_counts", C.c_int32),
        ("pad_", C.c_int32),
    ]


class MetricsC(C.Structure):
    _fields_ = [
        ("passes", C.c_uint64),
        ("sparse_passes", C.c_uint64),
        ("dense_passes", C.c_uint64),
        ("recovery_passes", C.c_uint64),
        ("pages_transferred", C.c_uint64),
        ("bytes_transferred", C.c_uint64),
        ("update_attempts", C.c_uint64),
        ("valid_updates", C.c_uint64),
        ("skipped_vertices", C.c_uint64),
        ("edges_read", C.c_uint64),
        ("virtual_makespan", C.c_double),
        ("wall_seconds", C.c_double),
        ("has_prediction_accuracy", C.c_int32),
        ("pad_", C.c_int32),
        ("prediction_accuracy", C.c_double),
        ("device_seconds", C.c_double),
        ("upload_seconds", C.c_double),
        ("kernel_launches", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("kernel_runs", C.c_uint64),
        ("relax_seconds", C.c_double),
        ("relax_launches", C.c_uint64),
        ("gathers", C.c_uint64),
        ("edges_streamed", C.c_uint64),
        ("dest_visits", C.c_uint64),
    ]


class TraceEventC(C.Structure):
    _fields_ = [
        ("time", C.c_double),
        ("kind", C.c_int32),
        ("page_id", C.c_uint32),
        ("pass_index", C.c_uint32),
        ("pad_", C.c_uint32),
    ]


class DeviceInfo(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("sm_count", C.c_int32),
        ("l2_bytes", C.c_int32),
        ("cc_major", C.c_int32),
        ("cc_minor", C.c_int32),
        ("pad_", C.c_int32),
        ("total_mem", C.c_uint64),
        ("free_mem", C.c_uint64),
        ("name", C.c_char * 64),
    ]


class GraphSpec(C.Structure):
    _fields_ = [
        ("scale", C.c_int32),
        ("edge_factor", C.c_uint32),
        ("a", C.c_double),
        ("b", C.c_double),
        ("c", C.c_double),
        ("d", C.c_double),
        ("seed", C.c_uint64),
        ("weight_lo", C.c_uint32),
        ("weight_hi", C.c_uint32),
        ("weight_seed", C.c_uint64),
        ("symmetrize", C.c_int32),
        ("page_vertex_capacity", C.c_uint32),
    ]


class GraphInfo(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_uint32),
        ("num_pages", C.c_uint32),
        ("num_edges", C.c_uint64),
        ("page_vertex_capacity", C.c_uint32),
        ("weighted", C.c_int32),
        ("has_csr_edges", C.c_int32),
        ("csr_weighted", C.c_int32),
        ("csr_derived", C.c_int32),
        ("adjacency_on_host", C.c_int32),
    ]


BUILD_CSR_EDGES = 1
EXCHANGE_PEER = 1

# Every symbol include/seraph.h declares: (name, restype, argtypes)
_VP, _U32, _U64, _I32, _D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
SIGNATURES = {
    "sr_abi_version": (C.c_int, []),
    "sr_default_config": (None, [C.POINTER(RunConfig)]),
    "sr_global_error": (C.c_char_p, []),
    "sr_open": (C.c_int, [C.c_int, _U64, C.POINTER(_VP)]),
    "sr_close": (None, [_VP]),
    "sr_last_error": (C.c_char_p, [_VP]),
    "sr_device_query": (C.c_int, [C.c_int, C.POINTER(DeviceInfo)]),
    "sr_load_csr": (C.c_int, [_VP, _U32, _U64, _VP, _VP, _VP]),
    "sr_load_pages": (C.c_int, [_VP, _U32, _U32, C.c_int, C.POINTER(PageView), _U32]),
    "sr_loaded_page_bytes": (_U64, [_VP]),
    "sr_run": (C.c_int, [_VP, C.POINTER(RunConfig), _VP, _VP, C.POINTER(MetricsC),
                         C.POINTER(PassStatsC), _U32, C.POINTER(_U32)]),
    "sr_run_graph": (C.c_int, [_VP, _U32, _U64, _VP, _VP, _VP, _U32, C.c_int, C.POINTER(PageView), _U32,
                               C.POINTER(RunConfig), _VP, _VP, C.POINTER(MetricsC),
                               C.POINTER(PassStatsC), _U32, C.POINTER(_U32)]),
    "sr_get_trace": (C.c_int, [_VP, C.POINTER(TraceEventC), _U64, C.POINTER(_U64)]),
    "sr_verify_fixpoint": (C.c_int, [_VP, C.c_int, _VP, C.POINTER(_U64)]),
    "sr_bench_pull_sweep": (C.c_int, [_VP, C.c_int, _U32, C.POINTER(_D), C.POINTER(_U64)]),
    "sr_build_graph": (C.c_int, [_VP, _U32, _U64, _VP, _VP, _VP, _U32, C.c_int]),
    "sr_generate_graph": (C.c_int, [_VP, C.POINTER(GraphSpec), C.c_int]),
    "sr_graph_info_get": (C.c_int, [_VP, C.POINTER(GraphInfo)]),
    "sr_load_srph": (C.c_int, [_VP, C.c_char_p, _U32, C.c_int]),
    "sr_export_graph": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "sr_rmat_generate_device": (C.c_int, [C.c_int, C.c_int, _U64, _D, _D, _D, _D, _U64, _VP, _VP,
                                          _U64, _U32, _U32, _VP]),
    "sr_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8 * 128)]),
    "sr_host_alloc": (C.c_int, [_U64, C.POINTER(_VP)]),
    "sr_host_free": (None, [_VP]),
    "sr_device_sync": (C.c_int, [C.c_int]),
    "sr_bench_h2d": (C.c_int, [C.c_int, _U64, _U32, C.POINTER(_D)]),
    "sr_flush_l2": (C.c_int, [_VP, _U64]),
    "sr_attach_world": (C.c_int, [_VP, C.c_int, C.c_int, C.POINTER(C.c_uint8 * 128)]),
    "sr_attach_loopback": (C.c_int, [_VP, C.c_int, C.c_int, C.c_char_p, C.c_int]),
    "sr_set_exchange": (C.c_int, [_VP, C.c_int]),
    "sr_group_open": (C.c_int, [C.POINTER(C.c_int), C.c_int, _U64, C.c_int, C.POINTER(_VP)]),
    "sr_group_close": (None, [_VP]),
    "sr_group_last_error": (C.c_char_p, [_VP]),
    "sr_group_size": (C.c_int, [_VP]),
    "sr_group_load_graph": (C.c_int, [_VP, _U32, _U64, _VP, _VP, _VP, _U32, C.c_int,
                                      C.POINTER(PageView), _U32, C.c_int]),
    "sr_group_run": (C.c_int, [_VP, C.POINTER(RunConfig), _VP, _VP, C.POINTER(MetricsC),
                               C.POINTER(PassStatsC), _U32, C.POINTER(_U32)]),
    "sr_group_run_graph": (C.c_int, [_VP, _U32, _U64, _VP, _VP, _VP, _U32, C.c_int,
                                     C.POINTER(PageView), _U32, C.POINTER(RunConfig), _VP, _VP,
                                     C.POINTER(MetricsC), C.POINTER(PassStatsC), _U32,
                                     C.POINTER(_U32)]),
    "sr_group_graph_info": (C.c_int, [_VP, C.c_int, C.POINTER(GraphInfo)]),
    "sr_shard_plan": (C.c_int, [_U32, _VP, _U32, _VP]),
    "sr_rmat_generate": (C.c_int, [C.c_int, _U64, _D, _D, _D, _D, _U64, _VP, _VP, C.c_int]),
    "sr_weights_generate": (C.c_int, [_U64, _U64, _U32, _U32, _VP, C.c_int]),
    "sr_build_csr": (C.c_int, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
    "sr_build_csc": (C.c_int, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
    "sr_page_offsets": (C.c_int, [_U32, _U32, _VP, _VP]),
    "sr_out_offsets": (C.c_int, [_U32, _U64, _VP, _VP, C.c_int]),
    "sr_symmetrize": (C.c_int, [_U64, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libseraph.so not found at {LIB_PATH}: build it with `make lib` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int, ctx=None, group=None) -> None:
    if rc == SR_OK:
        return
    if group is not None:
        msg = lib.sr_group_last_error(group)
    else:
        msg = lib.sr_last_error(ctx) if ctx else lib.sr_global_error()
    text = msg.decode() if msg else f"error {rc}"
    raise _CODES.get(rc, Error)(text)


def default_config() -> RunConfig:
    c = RunConfig()
    lib.sr_default_config(C.byref(c))
    return c


def ptr(a) -> int | None:
    """Address of a contiguous numpy array (None for empty/None)."""
    if a is None or a.size == 0:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to libseraph must be contiguous"
    return a.ctypes.data


class PinnedArena:
    """Page-locked host arrays from sr_host_alloc (freed with the arena)."""

    def __init__(self):
        self._bufs = []

    def array(self, n: int, dtype) -> "np.ndarray":
        import numpy as np
        dt = np.dtype(dtype)
        nbytes = max(int(n) * dt.itemsize, 1)
        p = C.c_void_p()
        check(lib.sr_host_alloc(nbytes, C.byref(p)))
        self._bufs.append(p.value)
        buf = (C.c_uint8 * nbytes).from_address(p.value)
        return np.frombuffer(buf, dtype=dt, count=int(n))

    def close(self):
        for p in self._bufs:
            lib.sr_host_free(p)
        self._bufs = []

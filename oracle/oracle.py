"""TEST INFRASTRUCTURE ONLY -- ctypes access to the parity oracles.

* ``liboracle.so``: plain-C restatement of the reference algorithms
  (seraph_oracle.c; every function cites the reference file:line it follows).
* ``_ref/libpagestream_ref.so`` (optional): the unmodified reference library
  compiled from /root/reference by ``make -C oracle ref``.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module; the product never does.
Parity status: BFS/CC/SSSP pinned (generator, builders and solvers are checked
against the reference itself and its golden vectors); PageRank parity
unpinned (no reference implementation exists) -- its conventions are pinned by
known-answer tests instead.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_VP, _U32, _U64, _D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double
UNREACHED = 0xFFFFFFFF


def _p(a):
    if a is None or a.size == 0:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _load_oracle():
    path = os.path.join(_HERE, "liboracle.so")
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `make -C oracle`")
    lib = C.CDLL(path)
    sig = {
        "oracle_generate_rmat": (C.c_int, [C.c_int, _U64, _D, _D, _D, _U64, _VP, _VP]),
        "oracle_assign_weights": (C.c_int, [_U64, _U64, _U32, _U32, _VP]),
        "oracle_mix64": (_U64, [_U64]),
        "oracle_symmetrize": (None, [_U64, _VP, _VP, _VP, _VP, _VP, _VP]),
        "oracle_build_csr": (None, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP]),
        "oracle_build_csc": (None, [_U32, _U64, _VP, _VP, _VP, _U32, _VP, _VP, _VP, _VP]),
        "oracle_bfs": (None, [_U32, _VP, _VP, _U32, _VP]),
        "oracle_cc": (None, [_U32, _VP, _VP, _VP]),
        "oracle_sssp": (None, [_U32, _VP, _VP, _VP, _U32, _VP]),
        "oracle_brute_fixpoint": (None, [_U32, _U64, _VP, _VP, _VP, C.c_int, _U32, _VP]),
        "oracle_pagerank": (None, [_U32, _VP, _VP, _VP, _U32, _D, _VP]),
        "oracle_mt64_nth": (_U64, [_U64, _U64]),
        # oracle_par.c (OpenMP)
        "oracle_generate_rmat_par": (C.c_int, [C.c_int, _U64, _D, _D, _D, _U64, _VP, _VP, C.c_int]),
        "oracle_assign_weights_par": (C.c_int, [_U64, _U64, _U32, _U32, _VP, C.c_int]),
        "oracle_symmetrize_par": (None, [_U64, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
        "oracle_build_adjacency_par": (C.c_int, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
        "oracle_pagerank_par": (None, [_U32, _VP, _VP, _VP, _U32, _D, _VP, C.c_int]),
        "oracle_pr_compare": (None, [_U32, _VP, _VP, _D, _VP, C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


lib = _load_oracle()


def generate_rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, d=0.05, seed=0):
    """ingest.cpp:112-141, bit-exact (mt19937_64)."""
    m = (1 << scale) * edge_factor
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    rc = lib.oracle_generate_rmat(scale, edge_factor, a, b, c, seed, _p(src), _p(dst))
    assert rc == 0
    return src, dst


def generate_rmat_par(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, d=0.05, seed=0, threads=0):
    """generate_rmat on `threads` OpenMP threads (jump-ahead chunks), bit-exact."""
    m = (1 << scale) * edge_factor
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    assert lib.oracle_generate_rmat_par(scale, edge_factor, a, b, c, seed, _p(src), _p(dst),
                                        threads) == 0
    return src, dst


def assign_weights_par(m, seed, lo=1, hi=64, threads=0):
    w = np.empty(m, np.uint32)
    assert lib.oracle_assign_weights_par(m, seed, lo, hi, _p(w), threads) == 0
    return w


def symmetrize_par(src, dst, w=None, threads=0):
    m = src.size
    os_, od = np.empty(2 * m, np.uint32), np.empty(2 * m, np.uint32)
    ow = np.empty(2 * m, np.uint32) if w is not None and w.size else None
    lib.oracle_symmetrize_par(m, _p(src), _p(dst), _p(w) if ow is not None else None, _p(os_),
                              _p(od), _p(ow), threads)
    return os_, od, ow


def build_adjacency_par(n, key, other, w=None, threads=0):
    """Stable counting sort by key: (offsets u64[n+1], other, w) -- build_csr with
    key=src, the global CSC of build_csc_pages with key=dst."""
    m = key.size
    off = np.zeros(n + 1, np.uint64)
    oo = np.empty(m, np.uint32)
    ow = np.empty(m, np.uint32) if w is not None and w.size else None
    assert lib.oracle_build_adjacency_par(n, m, _p(key), _p(other),
                                          _p(w) if ow is not None else None, _p(off), _p(oo),
                                          _p(ow), threads) == 0
    return off, oo, ow


def pagerank_par(n, in_off, in_src, out_off, iters=20, damping=0.85, threads=0):
    """fp64 PageRank checker over a global CSC + CSR offsets (OpenMP)."""
    r = np.empty(n, np.float64)
    lib.oracle_pagerank_par(n, _p(in_off), _p(in_src), _p(out_off), iters, damping, _p(r), threads)
    return r


def pr_compare(got_f32, want_f64, rel_floor=1e-12, threads=0):
    """(max |d|, max |d|/want over want > rel_floor, sum |d|)."""
    out = np.zeros(3, np.float64)
    lib.oracle_pr_compare(want_f64.size, _p(np.ascontiguousarray(got_f32, np.float32)),
                          _p(want_f64), rel_floor, _p(out), threads)
    return float(out[0]), float(out[1]), float(out[2])


def assign_weights(m, seed, lo=1, hi=64):
    w = np.empty(m, np.uint32)
    assert lib.oracle_assign_weights(m, seed, lo, hi, _p(w)) == 0
    return w


def mt64_nth(seed: int, nth: int) -> int:
    return int(lib.oracle_mt64_nth(seed, nth))


def mix64(x: int) -> int:
    return int(lib.oracle_mix64(x))


def symmetrize(src, dst, w=None):
    m = src.size
    os_, od = np.empty(2 * m, np.uint32), np.empty(2 * m, np.uint32)
    ow = np.empty(2 * m, np.uint32) if w is not None and w.size else None
    lib.oracle_symmetrize(m, _p(src), _p(dst), _p(w) if ow is not None else None, _p(os_),
                          _p(od), _p(ow))
    return os_, od, ow


def build_csr(n, src, dst, w=None):
    m = src.size
    off = np.zeros(n + 1, np.uint64)
    nbr = np.empty(m, np.uint32)
    ow = np.empty(m, np.uint32) if w is not None and w.size else None
    lib.oracle_build_csr(n, m, _p(src), _p(dst), _p(w) if ow is not None else None, _p(off),
                         _p(nbr), _p(ow))
    return off, nbr, ow


def build_csc(n, src, dst, w, cap):
    """Global CSC + page-local offsets (|V| + P entries)."""
    m = src.size
    npg = (n + cap - 1) // cap
    off = np.zeros(n + 1, np.uint64)
    isrc = np.empty(m, np.uint32)
    iw = np.empty(m, np.uint32) if w is not None and w.size else None
    local = np.empty(n + npg, np.uint32)
    lib.oracle_build_csc(n, m, _p(src), _p(dst), _p(w) if iw is not None else None, cap, _p(off),
                         _p(isrc), _p(iw), _p(local))
    return off, isrc, iw, local


def solve(n, src, dst, w, algo: int, source: int = 0):
    """reference_solve (reference.cpp:77-90): 0 BFS, 1 CC, 2 SSSP."""
    off, nbr, ow = build_csr(n, src, dst, w)
    out = np.empty(n, np.uint32)
    if algo == 0:
        lib.oracle_bfs(n, _p(off), _p(nbr), source, _p(out))
    elif algo == 1:
        lib.oracle_cc(n, _p(off), _p(nbr), _p(out))
    else:
        lib.oracle_sssp(n, _p(off), _p(nbr), _p(ow), source, _p(out))
    return out


def solve_csr(algo, n, off, nbr, w=None, source=0):
    out = np.empty(n, np.uint32)
    if algo == 0:
        lib.oracle_bfs(n, _p(off), _p(nbr), source, _p(out))
    elif algo == 1:
        lib.oracle_cc(n, _p(off), _p(nbr), _p(out))
    else:
        lib.oracle_sssp(n, _p(off), _p(nbr), _p(w), source, _p(out))
    return out


def brute_fixpoint(n, src, dst, w, algo, source=0):
    out = np.empty(n, np.uint32)
    lib.oracle_brute_fixpoint(n, src.size, _p(src), _p(dst), _p(w) if w is not None else None,
                              algo, source, _p(out))
    return out


def pagerank(n, src, dst, iters=20, damping=0.85):
    """fp64 PageRank oracle (conventions: DESIGN.md §2)."""
    in_off, isrc, _, _ = build_csc(n, src, dst, None, max(n, 1))
    out_off, _, _ = build_csr(n, src, dst, None)
    r = np.empty(n, np.float64)
    lib.oracle_pagerank(n, _p(in_off), _p(isrc), _p(out_off), iters, damping, _p(r))
    return r


# ---------------------------------------------------------------------------
# The reference itself (optional; built here from /root/reference)
# ---------------------------------------------------------------------------
REF_PATH = os.path.join(_HERE, "_ref", "libpagestream_ref.so")


def load_reference():
    """Returns the reference library or None when it was not built."""
    if not os.path.exists(REF_PATH):
        return None
    ref = C.CDLL(REF_PATH)
    sig = {
        "ref_error": (C.c_char_p, []),
        "ref_generate_rmat": (C.c_int, [C.c_int, _U64, _D, _D, _D, _D, _U64, _VP, _VP]),
        "ref_assign_weights": (C.c_int, [_U32, _U64, _VP, _VP, _U64, _U32, _U32, _VP]),
        "ref_build_csr": (C.c_int, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP]),
        "ref_save_binary": (C.c_int, [_U32, _U64, _VP, _VP, _VP, C.c_char_p]),
        "ref_build_csc_pages": (C.c_int, [_U32, _U64, _VP, _VP, _VP, _U32, _VP, _VP, _VP]),
        "ref_reference_solve": (C.c_int, [_U32, _U64, _VP, _VP, _VP, C.c_int, _U32, _VP]),
        "ref_prepare": (_VP, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP, _U32]),
        "ref_release": (None, [_VP]),
        "ref_run_prepared": (C.c_int, [_VP, C.c_int, _U32, C.c_int, C.c_int, C.c_int, C.c_int,
                                       _U32, C.c_int, C.c_int, C.c_int, _D, _VP, _VP]),
        "ref_run": (C.c_int, [_U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP, _U32, C.c_int, _U32,
                              C.c_int, C.c_int, C.c_int, C.c_int, _U32, C.c_int, C.c_int,
                              C.c_int, _D, _VP, _VP]),
    }
    for name, (res, args) in sig.items():
        f = getattr(ref, name)
        f.restype, f.argtypes = res, args
    return ref


def ref_run(ref, n, out_off, out_nbr, out_w, in_off, in_src, in_w, cap, algo, source=0,
            predictor=0, schedule=0, mrt=2, reps=3, window=8, workers=4, clock=1, execution=0,
            density=0.05):
    """The reference engine's run() (engine.cpp:421-433); returns (values, metrics dict)."""
    vals = np.empty(n, np.uint32)
    met = np.zeros(16, np.float64)
    rc = ref.ref_run(n, out_nbr.size, _p(out_off), _p(out_nbr), _p(out_w), _p(in_off),
                     _p(in_src), _p(in_w), cap, algo, source, predictor, schedule, mrt, reps,
                     window, workers, clock, execution, density, _p(vals), _p(met))
    if rc != 0:
        raise RuntimeError(ref.ref_error().decode())
    keys = ["passes", "sparse_passes", "dense_passes", "recovery_passes", "pages_transferred",
            "bytes_transferred", "update_attempts", "valid_updates", "skipped_vertices",
            "edges_read", "virtual_makespan", "wall_seconds", "has_accuracy", "accuracy"]
    return vals, dict(zip(keys, met[:14].tolist()))


_REF_KEYS = ["passes", "sparse_passes", "dense_passes", "recovery_passes", "pages_transferred",
             "bytes_transferred", "update_attempts", "valid_updates", "skipped_vertices",
             "edges_read", "virtual_makespan", "wall_seconds", "has_accuracy", "accuracy"]


class RefGraph:
    """The reference's CsrGraph + PageSet built once from flat arrays (same layouts)."""

    def __init__(self, ref, n, out_off, out_nbr, out_w, in_off, in_src, in_w, cap):
        self.ref = ref
        self.n = n
        self.h = ref.ref_prepare(n, out_nbr.size, _p(out_off), _p(out_nbr), _p(out_w),
                                 _p(in_off), _p(in_src), _p(in_w), cap)
        if not self.h:
            raise RuntimeError(ref.ref_error().decode())

    def run(self, algo, source=0, predictor=0, schedule=0, mrt=2, reps=3, window=8, workers=4,
            clock=1, execution=0, density=0.05, want_values=False):
        vals = np.empty(self.n, np.uint32) if want_values else None
        met = np.zeros(16, np.float64)
        rc = self.ref.ref_run_prepared(self.h, algo, source, predictor, schedule, mrt, reps,
                                       window, workers, clock, execution, density, _p(vals),
                                       _p(met))
        if rc != 0:
            raise RuntimeError(self.ref.ref_error().decode())
        return vals, dict(zip(_REF_KEYS, met[:14].tolist()))

    def close(self):
        if self.h:
            self.ref.ref_release(self.h)
            self.h = None

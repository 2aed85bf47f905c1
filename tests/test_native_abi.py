"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/seraph.h declares, and its host-side logic (builders, generator,
shard plan, error mapping) is correct.  No kernel is launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_1806_00762_b200 import _native as N
from paper_1806_00762_b200 import pagestream as ps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "seraph.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sr_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(N.lib, s), s
        assert s in N.SIGNATURES, f"{s} not bound in _native.py"
    assert N.lib.sr_abi_version() == 1


def test_default_config_matches_reference_defaults():  # engine.hpp:39-52, scheduler.hpp:19-47
    c = N.default_config()
    assert c.window_capacity == 8 and c.max_reentry_times == 2 and c.buffer_repetitions == 3
    assert c.density_threshold_fraction == 0.05 and c.worker_count == 4
    assert c.bytes_per_time_unit == 11.0 and c.edges_per_time_unit_per_worker == 1.75
    assert c.clock == N.CLOCK_VIRTUAL and c.predictor == N.PRED_OFF


def test_struct_layouts_match_header_sizes():
    assert C.sizeof(N.PageView) == 40
    assert C.sizeof(N.PassStatsC) == 4 + 4 + 8 * 5 + 8 * 6 + 8
    assert C.sizeof(N.TraceEventC) == 24


def test_open_without_device_raises_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(N.CudaError):
        ps.Engine(0)


@pytest.mark.parametrize("weighted", [False, True])
def test_host_builders_equal_oracle_random(weighted):  # test_graph.cpp:113-140
    rng = np.random.default_rng(12345)
    for _ in range(40):
        n = int(rng.integers(1, 25))
        m = int(rng.integers(0, 61))
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = rng.integers(0, n, m).astype(np.uint32)
        w = rng.integers(1, 17, m).astype(np.uint32) if weighted else np.zeros(0, np.uint32)
        el = ps.EdgeList(n, src, dst, w)
        csr = ps.build_csr(el, threads=3)
        off, nbr, ow = O.build_csr(n, src, dst, w if weighted else None)
        assert np.array_equal(csr.out_offsets, off) and np.array_equal(csr.out_neighbors, nbr)
        if weighted:
            assert np.array_equal(csr.out_weights, ow)
        for cap in (1, 3, 7, 64):
            pages = ps.build_csc_pages(el, cap, threads=2)
            _, isrc, iw, local = O.build_csc(n, src, dst, w if weighted else None, cap)
            assert np.array_equal(np.concatenate([p.in_offsets for p in pages.pages]), local)
            got = np.concatenate([p.in_sources for p in pages.pages]) if m else np.zeros(0)
            assert np.array_equal(got, isrc)
            total = sum(ps.page_bytes(p, weighted) for p in pages.pages)
            assert total == ((n + pages.page_count()) + m * (2 if weighted else 1)) * 4
            cov = np.zeros(n, int)
            for p in pages.pages:
                assert p.vertex_begin < p.vertex_end
                cov[p.vertex_begin:p.vertex_end] += 1
            assert (cov == 1).all()


def test_build_csr_large_stable_against_oracle():
    src, dst = O.generate_rmat(14, 16, seed=9)
    w = O.assign_weights(src.size, 4)
    el = ps.EdgeList(1 << 14, src, dst, w)
    csr = ps.build_csr(el, threads=8)
    off, nbr, ow = O.build_csr(1 << 14, src, dst, w)
    assert np.array_equal(csr.out_offsets, off) and np.array_equal(csr.out_neighbors, nbr)
    assert np.array_equal(csr.out_weights, ow)


def test_graph_contract_errors():  # test_graph.cpp:27-34, :84-88
    with pytest.raises(ps.InputError):
        ps.build_csr(ps.EdgeList.from_pairs(2, [(2, 0)]))
    with pytest.raises(ps.InputError):
        ps.build_csr(ps.EdgeList.from_pairs(2, [(0, 5)]))
    with pytest.raises(ps.ConfigError):
        ps.build_csc_pages(ps.EdgeList.from_pairs(1, []), 0)
    with pytest.raises(ps.ConfigError):
        ps.make_bfs(3, 3)
    with pytest.raises(ps.ConfigError):
        ps.make_sssp(0, 3, False)


def test_symmetrize_and_goldens():  # test_graph.cpp:94-111
    sym = ps.symmetrize(ps.EdgeList.from_pairs(3, [(0, 1), (1, 2)], [7, 9]))
    got = sorted(zip(sym.src.tolist(), sym.dst.tolist(), sym.weights.tolist()))
    assert got == [(0, 1, 7), (1, 0, 7), (1, 2, 9), (2, 1, 9)]
    pages = ps.build_csc_pages(ps.EdgeList.from_pairs(10, []), 4)
    assert [(p.vertex_begin, p.vertex_end) for p in pages.pages] == [(0, 4), (4, 8), (8, 10)]
    assert ps.resolve_page_capacity(0, 4096) == 128 and ps.resolve_page_capacity(0, 5) == 1


def test_fast_rmat_law_and_determinism():
    a = ps.generate_rmat_fast(12, 16, seed=3, threads=4)
    b = ps.generate_rmat_fast(12, 16, seed=3, threads=7)
    assert np.array_equal(a.src, b.src) and np.array_equal(a.dst, b.dst)
    # the reference's own stream (generate_rmat, ingest.cpp:112-141)
    s, d = O.generate_rmat(12, 16, seed=3)
    assert np.array_equal(a.src, s) and np.array_equal(a.dst, d)
    w = ps.assign_weights_fast(a, 11, 1, 64, threads=5).weights
    assert np.array_equal(w, O.assign_weights(a.num_edges(), 11, 1, 64))
    assert a.num_edges() == 16 * 4096 and int(a.src.max()) < 4096
    # quadrant law: P(top bit of dst set) = b + d = 0.24
    frac = float(((a.dst >> 11) & 1).mean())
    assert abs(frac - 0.24) < 0.01
    u = ps.generate_rmat_fast(12, 16, 0.25, 0.25, 0.25, 0.25, seed=1)
    assert abs(float(((u.src >> 11) & 1).mean()) - 0.5) < 0.01


def test_shard_plan_edge_balanced():
    src, dst = O.generate_rmat(12, 16, seed=0)
    in_off, _, _, _ = O.build_csc(4096, src, dst, None, 4096)
    for parts in (1, 2, 4, 8):
        cuts = ps.shard_plan(4096, in_off, parts)
        assert cuts[0] == 0 and cuts[-1] == 4096 and (np.diff(cuts.astype(int)) >= 0).all()
        loads = np.diff(in_off[cuts.astype(np.int64)].astype(np.int64))
        assert loads.max() <= src.size / parts + int(np.diff(in_off.astype(np.int64)).max())


def test_struct_sizes_match_compiled_header(tmp_path):
    """ctypes mirrors of the C-ABI structs have the compiler's sizes."""
    import subprocess
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "seraph.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(sr_page_view),sizeof(sr_run_config),sizeof(sr_pass_stats),'
                   'sizeof(sr_metrics),sizeof(sr_trace_event),sizeof(sr_device_info));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [C.sizeof(t) for t in (N.PageView, N.RunConfig, N.PassStatsC, N.MetricsC,
                                  N.TraceEventC, N.DeviceInfo)]
    assert got == want

"""The oracle pinned against the reference: golden fixtures produced by the
reference compiled from its own sources (tests/golden/make_golden.py), the
reference's inline known answers (test_algorithms.cpp, test_bench.cpp,
test_graph.cpp) and the C++ standard's mt19937_64 check value.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["rmat_s8_ef16_seed3", "rmat_s10_ef16_seed0", "rmat_s12_ef8_seed1"]


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def test_mt19937_64_standard_check_value():
    # [rand.predef]: 10000th output of default-seeded mt19937_64
    assert O.mt64_nth(5489, 10000) == 9981545732273789042


@pytest.mark.parametrize("name", CASES)
def test_generator_weights_builders_match_reference(name):
    g = load(name)
    scale = int(np.log2(int(g["n"][0])))
    ef = g["src"].size // int(g["n"][0])
    seed = int(name.split("seed")[1])
    src, dst = O.generate_rmat(scale, ef, seed=seed)
    assert np.array_equal(src, g["src"]) and np.array_equal(dst, g["dst"])
    w = O.assign_weights(src.size, O.mix64(seed ^ 0x77), 1, 64)
    assert np.array_equal(w, g["w"])
    n = int(g["n"][0])
    off, nbr, ow = O.build_csr(n, src, dst, w)
    assert np.array_equal(off, g["csr_off"]) and np.array_equal(nbr, g["csr_nbr"])
    assert np.array_equal(ow, g["csr_w"])
    cap = int(g["cap"][0])
    _, isrc, iw, local = O.build_csc(n, src, dst, w, cap)
    assert np.array_equal(local, g["page_local"]) and np.array_equal(isrc, g["page_src"])
    assert np.array_equal(iw, g["page_w"])


@pytest.mark.parametrize("name", CASES)
def test_solvers_match_reference_solve(name):
    g = load(name)
    n = int(g["n"][0])
    assert np.array_equal(O.solve(n, g["src"], g["dst"], g["w"], 0, 0), g["bfs"])
    assert np.array_equal(O.solve(n, g["src"], g["dst"], g["w"], 2, 0), g["sssp"])
    ss, sd, _ = O.symmetrize(g["src"], g["dst"])
    assert np.array_equal(O.solve(n, ss, sd, None, 1), g["cc"])


def test_uniform_quadrants_cc():
    g = load("uniform_s10_seed5")
    src, dst = O.generate_rmat(10, 16, 0.25, 0.25, 0.25, 0.25, seed=5)
    assert np.array_equal(src, g["src"]) and np.array_equal(dst, g["dst"])
    ss, sd, _ = O.symmetrize(src, dst)
    assert np.array_equal(O.solve(1024, ss, sd, None, 1), g["cc"])


def test_reference_runs_values_equal_oracle():
    with open(os.path.join(GOLD, "ref_runs_s7.json")) as fh:
        d = json.load(fh)
    src, dst = O.generate_rmat(7, 8, seed=11)
    want = O.solve(128, src, dst, None, 0, 0)
    for key, run in d["runs"].items():
        assert np.array_equal(np.array(run["values"], np.uint32), want), key
        assert run["metrics"]["passes"] >= 1


# ---- reference inline goldens -------------------------------------------------
def _arr(x):
    return np.array(x, np.uint32)


def test_algorithm_goldens():  # test_algorithms.cpp:42-98, test_bench.cpp:15-31
    assert O.solve(3, _arr([0, 1]), _arr([1, 2]), None, 0, 0).tolist() == [0, 1, 2]
    out = O.solve(3, _arr([0]), _arr([1]), None, 0, 0).tolist()
    assert out == [0, 1, O.UNREACHED]
    ss, sd, _ = O.symmetrize(_arr([0, 2]), _arr([1, 3]))
    assert O.solve(4, ss, sd, None, 1).tolist() == [0, 0, 2, 2]
    ss, sd, _ = O.symmetrize(_arr([0, 1, 2, 3, 4]), _arr([1, 2, 3, 4, 5]))
    assert O.solve(6, ss, sd, None, 1).tolist() == [0] * 6
    assert O.solve(3, _arr([]), _arr([]), None, 1).tolist() == [0, 1, 2]
    assert O.solve(3, _arr([0, 0, 2]), _arr([1, 2, 1]), _arr([5, 1, 2]), 2, 0).tolist() == [0, 3, 1]


def test_brute_force_fixpoint_agrees_random():  # test_bench.cpp:33-47
    rng = np.random.default_rng(17)
    for _ in range(30):
        n = int(rng.integers(1, 21))
        m = int(rng.integers(0, 61))
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = rng.integers(0, n, m).astype(np.uint32)
        w = rng.integers(1, 17, m).astype(np.uint32)
        s = int(rng.integers(0, n))
        assert np.array_equal(O.solve(n, src, dst, w, 0, s), O.brute_fixpoint(n, src, dst, w, 0, s))
        assert np.array_equal(O.solve(n, src, dst, w, 2, s), O.brute_fixpoint(n, src, dst, w, 2, s))
        ss, sd, _ = O.symmetrize(src, dst)
        assert np.array_equal(O.solve(n, ss, sd, None, 1), O.brute_fixpoint(n, ss, sd, None, 1))


def test_csr_csc_goldens():  # test_graph.cpp:13-63
    off, nbr, _ = O.build_csr(3, _arr([0, 0, 1]), _arr([1, 2, 2]))
    assert off.tolist() == [0, 2, 3, 3] and nbr.tolist() == [1, 2, 2]
    _, isrc, _, local = O.build_csc(4, _arr([0, 2, 1]), _arr([1, 1, 3]), None, 2)
    assert local.tolist() == [0, 0, 2, 0, 0, 1]
    assert isrc.tolist() == [0, 2, 1]


# ---- PageRank oracle: known answers (no reference implementation exists) ------
def test_pagerank_oracle_known_answers():
    r = O.pagerank(3, _arr([0, 1, 2]), _arr([1, 2, 0]), 20, 0.85)
    assert np.allclose(r, 1 / 3, atol=1e-15)
    d = 0.85
    r = O.pagerank(2, _arr([0]), _arr([1]), 20, d)
    assert abs(r[0] - (1 - d) / 2) < 1e-15
    assert abs(r[1] - ((1 - d) / 2 + d * (1 - d) / 2)) < 1e-15
    # star: leaves 1..4 -> 0; dangling mass of 0 dropped
    r = O.pagerank(5, _arr([1, 2, 3, 4]), _arr([0, 0, 0, 0]), 20, d)
    leaf = (1 - d) / 5
    assert np.allclose(r[1:], leaf) and abs(r[0] - (leaf + d * 4 * leaf)) < 1e-15


# ---- multi-threaded oracle pipeline (oracle_par.c): equal to the sequential,
# reference-pinned restatements ---------------------------------------------------
@pytest.mark.parametrize("case", [(8, 16, 3, 1), (10, 16, 0, 7), (12, 8, 1, 3), (11, 3, 9, 16)])
def test_parallel_generator_equals_sequential(case):
    scale, ef, seed, threads = case
    for q in ((0.57, 0.19, 0.19, 0.05), (0.25, 0.25, 0.25, 0.25)):
        s1, d1 = O.generate_rmat(scale, ef, *q[:3], seed=seed)
        s2, d2 = O.generate_rmat_par(scale, ef, *q, seed=seed, threads=threads)
        assert np.array_equal(s1, s2) and np.array_equal(d1, d2)
    w1 = O.assign_weights(s1.size, seed + 1, 1, 64)
    assert np.array_equal(w1, O.assign_weights_par(s1.size, seed + 1, 1, 64, threads))


def test_parallel_generator_matches_reference_fixture():
    g = load("rmat_s10_ef16_seed0")
    src, dst = O.generate_rmat_par(10, 16, seed=0, threads=5)
    assert np.array_equal(src, g["src"]) and np.array_equal(dst, g["dst"])


@pytest.mark.parametrize("threads", [1, 4, 13])
def test_parallel_builders_equal_sequential(threads):
    rng = np.random.default_rng(threads)
    for n, m in ((1, 0), (7, 50), (3000, 40000), (70000, 300000)):
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = rng.integers(0, n, m).astype(np.uint32)
        w = rng.integers(1, 65, m).astype(np.uint32)
        off, nbr, ow = O.build_csr(n, src, dst, w)
        off2, nbr2, ow2 = O.build_adjacency_par(n, src, dst, w, threads)
        assert np.array_equal(off, off2) and np.array_equal(nbr, nbr2)
        assert m == 0 or np.array_equal(ow, ow2)
        ioff, isrc, iw, _ = O.build_csc(n, src, dst, w, max(n, 1))
        ioff2, isrc2, iw2 = O.build_adjacency_par(n, dst, src, w, threads)
        assert np.array_equal(ioff, ioff2) and np.array_equal(isrc, isrc2)
        ss, sd, sw = O.symmetrize(src, dst, w)
        ss2, sd2, sw2 = O.symmetrize_par(src, dst, w, threads)
        assert np.array_equal(ss, ss2) and np.array_equal(sd, sd2)


def test_parallel_pagerank_equals_sequential():
    src, dst = O.generate_rmat(12, 8, seed=2)
    n = 1 << 12
    want = O.pagerank(n, src, dst, 20, 0.85)
    ioff, isrc, _ = O.build_adjacency_par(n, dst, src)
    ooff, _, _ = O.build_adjacency_par(n, src, dst)
    got = O.pagerank_par(n, ioff, isrc, ooff, 20, 0.85, threads=6)
    assert np.max(np.abs(got - want)) < 1e-15
    mx, mr, l1 = O.pr_compare(got.astype(np.float32), want)
    assert mx < 1e-9 and mr < 1e-6 and l1 < 1e-6

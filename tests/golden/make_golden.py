"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference/proj/src).  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures are small .npz files committed to the repo; tests compare the
oracle restatement and the GPU engine against them on the GPU box, where the
reference sources are absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

ref = O.load_reference()
assert ref is not None, "build oracle/_ref first (make -C oracle ref)"


def p(a):
    return a.ctypes.data if a is not None and a.size else None


def ref_rmat(scale, ef, seed, a=0.57, b=0.19, c=0.19, d=0.05):
    m = (1 << scale) * ef
    src, dst = np.empty(m, np.uint32), np.empty(m, np.uint32)
    assert ref.ref_generate_rmat(scale, ef, a, b, c, d, seed, p(src), p(dst)) == 0
    return src, dst


def ref_weights(n, src, dst, seed, lo=1, hi=64):
    w = np.empty(src.size, np.uint32)
    assert ref.ref_assign_weights(n, src.size, p(src), p(dst), seed, lo, hi, p(w)) == 0
    return w


def ref_solve(n, src, dst, w, algo, source=0):
    out = np.empty(n, np.uint32)
    assert ref.ref_reference_solve(n, src.size, p(src), p(dst), p(w), algo, source, p(out)) == 0
    return out


def ref_csr(n, src, dst, w):
    off = np.empty(n + 1, np.uint64)
    nbr = np.empty(src.size, np.uint32)
    ow = np.empty(src.size, np.uint32)
    assert ref.ref_build_csr(n, src.size, p(src), p(dst), p(w), p(off), p(nbr), p(ow)) == 0
    return off, nbr, ow


def ref_pages(n, src, dst, w, cap):
    npg = (n + cap - 1) // cap
    local = np.empty(n + npg, np.uint32)
    isrc = np.empty(src.size, np.uint32)
    iw = np.empty(src.size, np.uint32)
    assert ref.ref_build_csc_pages(n, src.size, p(src), p(dst), p(w), cap, p(local), p(isrc),
                                   p(iw)) == 0
    return local, isrc, iw


def ref_run_virtual(n, src, dst, w, cap, algo, schedule, predictor, window=4):
    off, nbr, ow = ref_csr(n, src, dst, w)
    # global CSC offsets from the page-local ones
    local, isrc, iw = ref_pages(n, src, dst, w, cap)
    in_off = np.zeros(n + 1, np.uint64)
    npg = (n + cap - 1) // cap
    base = 0
    for pg in range(npg):
        vb, ve = pg * cap, min((pg + 1) * cap, n)
        loc = local[vb + pg: ve + pg + 1].astype(np.uint64)
        in_off[vb:ve + 1] = base + loc
        base += int(loc[-1])
    vals, met = O.ref_run(ref, n, off, nbr, ow if w is not None else None, in_off, isrc,
                          iw if w is not None else None, cap, algo, 0, predictor, schedule, 2,
                          3, window, 4, 0, 0, 0.05)
    return vals, met


def main():
    cases = {}
    # RMAT graphs of the configs' family at test scale (seed, weight seed = bench mix64 rule)
    for scale, ef, seed in [(8, 16, 3), (10, 16, 0), (12, 8, 1)]:
        n = 1 << scale
        src, dst = ref_rmat(scale, ef, seed)
        w = ref_weights(n, src, dst, O.mix64(seed ^ 0x77))
        ss = np.empty(2 * src.size, np.uint32)
        sd = np.empty(2 * src.size, np.uint32)
        ss[0::2], ss[1::2] = src, dst
        sd[0::2], sd[1::2] = dst, src
        cap = (n + 31) // 32
        off, nbr, ow = ref_csr(n, src, dst, w)
        local, isrc, iw = ref_pages(n, src, dst, w, cap)
        name = f"rmat_s{scale}_ef{ef}_seed{seed}"
        cases[name] = dict(
            n=np.array([n]), src=src, dst=dst, w=w,
            bfs=ref_solve(n, src, dst, w, 0), sssp=ref_solve(n, src, dst, w, 2),
            cc=ref_solve(n, ss, sd, None, 1), csr_off=off, csr_nbr=nbr, csr_w=ow,
            page_local=local, page_src=isrc, page_w=iw, cap=np.array([cap]))
    # uniform quadrants (config C4 family)
    src, dst = ref_rmat(10, 16, 5, 0.25, 0.25, 0.25, 0.25)
    n = 1 << 10
    ss = np.concatenate([np.stack([src, dst], 1).reshape(-1)])
    sym_src = np.empty(2 * src.size, np.uint32)
    sym_dst = np.empty(2 * src.size, np.uint32)
    sym_src[0::2], sym_src[1::2] = src, dst
    sym_dst[0::2], sym_dst[1::2] = dst, src
    cases["uniform_s10_seed5"] = dict(n=np.array([n]), src=src, dst=dst,
                                      cc=ref_solve(n, sym_src, sym_dst, None, 1))
    for name, arrays in cases.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    # reference run() in virtual mode: values + metrics (test_bench.cpp:104-131 spec)
    src, dst = ref_rmat(7, 8, 11)
    n = 128
    runs = {}
    # pipelined-fine with a predictor can livelock the reference (SURVEY §4,
    # scheduler.cpp:348-360): only predictor-off fine cells are recorded.
    for sched, pred in [(0, 0), (3, 2), (1, 1), (4, 0), (2, 0)]:
        vals, met = ref_run_virtual(n, src, dst, None, (n + 31) // 32, 0, sched, pred)
        runs[f"bfs_sched{sched}_pred{pred}"] = {"values": vals.tolist(), "metrics": met}
    with open(os.path.join(HERE, "ref_runs_s7.json"), "w") as fh:
        json.dump({"graph": {"scale": 7, "edge_factor": 8, "seed": 11}, "runs": runs}, fh)
    # mt19937_64 stream head (seed 0) as used by generate_rmat
    print("wrote", sorted(cases), "ref_runs_s7.json")


if __name__ == "__main__":
    main()

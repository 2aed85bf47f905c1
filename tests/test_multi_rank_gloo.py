"""world_size-2 CPU emulation (torch.distributed, gloo) of the sharded round
protocol that libseraph runs over NCCL (engine.cpp exchange_round):

  * destinations are cut into edge-balanced contiguous shards (sr_shard_plan);
  * a dense round relaxes only the rank's own destinations (pull), a sparse
    round pushes only from the rank's own frontier vertices;
  * the replicated value arrays are merged with an all-reduce MIN, and every
    rank derives the same next frontier from (merged < round snapshot), so all
    ranks take the same density-switch decision without further traffic.

The merged values must equal the oracle on every rank."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1806_00762_b200 import pagestream as ps

INF = np.uint64(0xFFFFFFFF)


def combine(algo, val, w):
    val = val.astype(np.uint64)
    if algo == 1:
        return val
    add = np.uint64(1) if algo == 0 else w.astype(np.uint64)
    out = val + add
    out[val == INF] = INF
    return np.minimum(out, INF)


def rank_main(rank, world, port, algo, scale, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1 << scale
    src, dst = O.generate_rmat(scale, 8, seed=3)
    w = O.assign_weights(src.size, 5)
    if algo == 1:
        src, dst, w = O.symmetrize(src, dst, w)
    in_off, in_src, in_w, _ = O.build_csc(n, src, dst, w, n)
    out_off, out_nbr, out_w = O.build_csr(n, src, dst, w)
    cuts = ps.shard_plan(n, in_off, world)
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    vals = np.full(n, INF, np.uint64)
    if algo == 1:
        vals = np.arange(n, dtype=np.uint64)
    else:
        vals[0] = 0
    changed = np.zeros(n, bool)
    changed[:] = algo == 1
    changed[0] = True
    m = src.size
    rounds = 0
    while changed.any():
        snap = vals.copy()
        out_edges = int((out_off[1:] - out_off[:-1])[changed].sum())
        if out_edges > 0.05 * m:  # density_switch (engine.cpp:56-61): dense pull, own dests
            e_lo, e_hi = int(in_off[lo]), int(in_off[hi])
            if e_hi > e_lo:
                cand = combine(algo, vals[in_src[e_lo:e_hi]], in_w[e_lo:e_hi])
                seg = in_off[lo:hi + 1].astype(np.int64) - e_lo
                nz = np.nonzero(seg[1:] > seg[:-1])[0]
                best = np.minimum.reduceat(cand, seg[:-1][nz])
                tgt = lo + nz
                vals[tgt] = np.minimum(vals[tgt], best)
        else:  # sparse push from the rank's own frontier vertices
            mine = np.nonzero(changed[lo:hi])[0] + lo
            for u in mine:
                a, b = int(out_off[u]), int(out_off[u + 1])
                if a == b:
                    continue
                cand = combine(algo, np.full(b - a, vals[u], np.uint64), out_w[a:b])
                np.minimum.at(vals, out_nbr[a:b].astype(np.int64), cand)
        t = torch.from_numpy(vals.astype(np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        vals = t.numpy().astype(np.uint64)
        changed = vals < snap
        rounds += 1
        assert rounds < 10000
    q.put((rank, vals.astype(np.uint32).tobytes(), rounds))
    dist.destroy_process_group()


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_two_rank_sharded_rounds_match_oracle(algo):
    scale = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29611 + algo
    procs = [ctx.Process(target=rank_main, args=(r, 2, port, algo, scale, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 1 << scale
    src, dst = O.generate_rmat(scale, 8, seed=3)
    w = O.assign_weights(src.size, 5)
    if algo == 1:
        s2, d2, _ = O.symmetrize(src, dst, w)
        want = O.solve(n, s2, d2, None, 1)
    else:
        want = O.solve(n, src, dst, w, algo, 0)
    outs = [np.frombuffer(b, np.uint32) for _, b, _ in sorted(res)]
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], want)

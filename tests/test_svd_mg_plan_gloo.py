"""CPU test of the multi-GPU SVD's host logic with
world_size 2 over gloo: each process owns the block-pair slots
mpjacobi_svd_mg_plan assigns to it (the same C++ code mpjacobi_svd_mg uses),
applies one sweep of one-sided block rotations [C_x C_y] <- [C_x C_y] U_k to
its slots' 32-column blocks only -- keeping a whole-size matrix whose other
blocks go stale, as the GPU path does -- and moves the blocks whose slot
changes rank with dist.send / dist.recv exactly as the plan's moves
prescribe; every block is then taken from its last owner and must equal the
same sweep applied to the whole matrix in one process.  No GPU: the 64 x 64
rotation blocks are seeded random orthogonal matrices, so this checks the
data movement (ownership, moves), not the Jacobi arithmetic (the emulated-rank
GPU tests check that bit for bit)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

BW, TW = 32, 64


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _u_block(r, k):
    rng = np.random.default_rng(5000 + 1000 * r + k)
    q, _ = np.linalg.qr(rng.standard_normal((TW, TW)))
    return q


def _cols(x, y):
    return np.r_[x * BW:(x + 1) * BW, y * BW:(y + 1) * BW]


def _start(np_, m=96):
    return np.random.default_rng(11).standard_normal((m, np_))


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2211_03339_b200 as mpj
    np_, pairs, moves = mpj.svd_mg_plan(n, world)
    mb = np_ // TW
    mbl = mb // world
    C = _start(np_)
    rounds = pairs.shape[0]
    for r in range(rounds):
        for kl in range(mbl):
            k = rank * mbl + kl
            c = _cols(*pairs[r, k])
            C[:, c] = C[:, c] @ _u_block(r, k)
        if r + 1 < rounds:
            reqs = []
            for blk, src, dst in moves[r]:
                if src == rank:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(C[:, blk * BW:(blk + 1) * BW])), dst))
            for blk, src, dst in moves[r]:
                if dst == rank:
                    buf = torch.empty((C.shape[0], BW), dtype=torch.float64)
                    dist.recv(buf, src)
                    C[:, blk * BW:(blk + 1) * BW] = buf.numpy()
            for q in reqs:
                q.wait()
    np.save(os.path.join(out_dir, f"C{rank}.npy"), C)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [256, 200, 512])
def test_svd_partition_two_ranks_gloo(tmp_path, n):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, str(tmp_path)), nprocs=world, join=True)
    import paper_2211_03339_b200 as mpj
    np_, pairs, moves = mpj.svd_mg_plan(n, world)
    mb = np_ // TW
    mbl = mb // world
    C = _start(np_)
    for r in range(pairs.shape[0]):           # single-process reference
        for k in range(mb):
            c = _cols(*pairs[r, k])
            C[:, c] = C[:, c] @ _u_block(r, k)
    last = pairs.shape[0] - 1
    Cs = [np.load(tmp_path / f"C{g}.npy") for g in range(world)]
    for k in range(mb):
        g = k // mbl
        for blk in pairs[last, k]:
            np.testing.assert_allclose(Cs[g][:, blk * BW:(blk + 1) * BW], C[:, blk * BW:(blk + 1) * BW], atol=1e-12)


def test_svd_plan_invariants():
    """Every round pairs all blocks; a block changes rank only when its slot
    does; moves are balanced (every rank sends as many blocks as it receives,
    so each keeps 2 mb / G blocks)."""
    import paper_2211_03339_b200 as mpj
    for n, G in ((512, 2), (1024, 4), (2048, 8), (300, 4)):
        np_, pairs, moves = mpj.svd_mg_plan(n, G)
        assert np_ % (64 * G) == 0 and np_ >= n
        mb = np_ // TW
        mbl = mb // G
        for r in range(pairs.shape[0]):
            assert sorted(pairs[r].ravel().tolist()) == list(range(2 * mb))
        for r, mv in enumerate(moves):
            own = {b: k // mbl for k in range(mb) for b in pairs[r, k]}
            nxt = {b: k // mbl for k in range(mb) for b in pairs[r + 1, k]}
            assert sorted((b, s, d) for b, s, d in mv) == sorted((b, own[b], nxt[b]) for b in own if own[b] != nxt[b])
            for g in range(G):
                assert sum(1 for _, s, _ in mv if s == g) == sum(1 for _, _, d in mv if d == g)

"""CPU test of the multi-GPU path's host logic with world_size 2
over gloo: each process owns the column blocks the library's partition plan
(mpjacobi_mg_plan, the same C++ code mpjacobi_eig_mg uses) assigns to it,
applies one sweep of block rotations T <- U^T T U, V <- V U to its columns --
all-gathering the rotation blocks and exchanging the boundary column blocks
with dist.send / dist.recv exactly as the plan prescribes -- and the gathered
result must equal the same sweep applied to the whole matrix in one process.
No GPU: the rotation blocks are seeded random orthogonal 64 x 64 matrices, so
the test checks the data movement (slots, physical positions, transfers), not
the Jacobi arithmetic (that is the GPU parity tests' job)."""
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
    rng = np.random.default_rng(1000 * r + k)
    q, _ = np.linalg.qr(rng.standard_normal((TW, TW)))
    return q


def _rows(top, bot):
    return np.r_[top * BW:(top + 1) * BW, bot * BW:(bot + 1) * BW]


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2211_03339_b200 as mpj
    np_, slots, xfers = mpj.mg_plan(n, world)
    mb = np_ // TW
    mbl = mb // world
    rng = np.random.default_rng(7)
    T = rng.standard_normal((np_, np_))
    T = 0.5 * (T + T.T)
    V = np.eye(np_)
    # initial layout: rank g holds global blocks 2 g mbl .. 2 (g+1) mbl - 1 at positions 0..2 mbl-1
    phys = [[2 * g * mbl + p for p in range(2 * mbl)] for g in range(world)]
    cols = lambda blk: np.arange(blk * BW, (blk + 1) * BW)
    Tl = np.concatenate([T[:, cols(b)] for b in phys[rank]], axis=1)
    Vl = np.concatenate([V[:, cols(b)] for b in phys[rank]], axis=1)
    for r in range(slots.shape[0]):
        # local rotation blocks, all-gathered in slot order
        mine = torch.from_numpy(np.stack([_u_block(r, rank * mbl + kl) for kl in range(mbl)]))
        allu = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allu, mine)
        U = torch.cat(allu).numpy()
        for kl in range(mbl):
            c = rank * mbl + kl
            top, bot, ptop, pbot = slots[r, c]
            lc = np.r_[ptop * BW:(ptop + 1) * BW, pbot * BW:(pbot + 1) * BW]
            for a in range(mb):
                ra = _rows(slots[r, a, 0], slots[r, a, 1])
                Tl[np.ix_(ra, lc)] = U[a].T @ Tl[np.ix_(ra, lc)] @ U[c]
            Vl[:, lc] = Vl[:, lc] @ U[c]
        # boundary block exchange, as prescribed by the plan
        sends = [x for x in xfers[r] if x[0] == rank]
        recvs = [x for x in xfers[r] if x[2] == rank]
        reqs = []
        for src, sp, dst, dp in sends:
            for M in (Tl, Vl):
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(M[:, sp * BW:(sp + 1) * BW])), dst))
        staged = []
        for src, sp, dst, dp in recvs:
            bufs = [torch.empty((np_, BW), dtype=torch.float64) for _ in range(2)]
            for b in bufs:
                dist.recv(b, src)
            staged.append((dp, bufs))
        for q in reqs:
            q.wait()
        for dp, (bt, bv) in staged:
            Tl[:, dp * BW:(dp + 1) * BW] = bt.numpy()
            Vl[:, dp * BW:(dp + 1) * BW] = bv.numpy()
        nphys = [p[:] for p in phys]
        for src, sp, dst, dp in xfers[r]:
            nphys[dst][dp] = phys[src][sp]
        phys = nphys
    np.save(os.path.join(out_dir, f"T{rank}.npy"), Tl)
    np.save(os.path.join(out_dir, f"V{rank}.npy"), Vl)
    np.save(os.path.join(out_dir, f"phys{rank}.npy"), np.array(phys[rank]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [256, 200])
def test_partition_plan_two_ranks_gloo(tmp_path, n):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, str(tmp_path)), nprocs=world, join=True)
    import paper_2211_03339_b200 as mpj
    np_, slots, xfers = mpj.mg_plan(n, world)
    mb = np_ // TW
    rng = np.random.default_rng(7)
    T = rng.standard_normal((np_, np_))
    T = 0.5 * (T + T.T)
    V = np.eye(np_)
    # single-process reference: the same block rotations on the whole matrix
    for r in range(slots.shape[0]):
        Ug = np.zeros((np_, np_))
        for k in range(mb):
            rk = _rows(slots[r, k, 0], slots[r, k, 1])
            Ug[np.ix_(rk, rk)] = _u_block(r, k)
        T = Ug.T @ T @ Ug
        V = V @ Ug
    # every global block must appear exactly once across the ranks
    blocks = []
    for g in range(world):
        Tl = np.load(tmp_path / f"T{g}.npy")
        Vl = np.load(tmp_path / f"V{g}.npy")
        phys = np.load(tmp_path / f"phys{g}.npy")
        for p, b in enumerate(phys):
            blocks.append(b)
            np.testing.assert_allclose(Tl[:, p * BW:(p + 1) * BW], T[:, b * BW:(b + 1) * BW], atol=1e-12)
            np.testing.assert_allclose(Vl[:, p * BW:(p + 1) * BW], V[:, b * BW:(b + 1) * BW], atol=1e-12)
    assert sorted(blocks) == list(range(np_ // BW))
    # one sweep of the merry-go-round returns the slots to their starting blocks
    assert [tuple(x) for x in slots[0, :, :2]] == [(2 * k, 2 * k + 1) for k in range(mb)]


def test_plan_invariants():
    """Plan shape: every round is a perfect matching of blocks into slots;
    transfers only between neighbouring ranks, at most 2 per rank boundary."""
    import paper_2211_03339_b200 as mpj
    for n, G in ((512, 2), (1024, 4), (1024, 8)):
        np_, slots, xfers = mpj.mg_plan(n, G)
        mb = np_ // TW
        for r in range(slots.shape[0]):
            blk = sorted(slots[r, :, :2].ravel().tolist())
            assert blk == list(range(2 * mb))
            for src, sp, dst, dp in xfers[r]:
                assert abs(src - dst) == 1
            assert len(xfers[r]) <= 2 * (G - 1)

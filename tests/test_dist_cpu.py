"""CPU, world_size-2 (gloo) check of the row-partitioned CG exchange pattern
(pk_dist.inc): group-aligned z-slabs, one-plane halo
exchange of the SpMV input, per-rank group partials at the local geometry,
ONE allgather of the partials, and the serial stage 2 on every rank -- the
gathered result must equal the single-process reduction bit for bit, and an
unaligned per-rank sum must not be relied on.  The oracle supplies the
arithmetic (test infrastructure); the communication is real torch.distributed
gloo traffic between two processes."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")
mp = pytest.importorskip("torch.multiprocessing")

from oracle import pk_oracle as orc  # noqa: E402

SIDE, GS, WORLD = 16, 64, 2  # n = 4096 = 64 groups of 64; slabs of 2048 rows = 8 planes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        a, _ = orc.poisson3d(SIDE)
        n, H = SIDE ** 3, SIDE * SIDE
        nloc = n // WORLD
        lo, hi = rank * nloc, (rank + 1) * nloc
        p = np.random.default_rng(7).random(n)  # the SpMV input every rank would hold locally
        # local haloed input: [H lower][nloc own][H upper]; halos come from the neighbours
        own = torch.from_numpy(p[lo:hi].copy())
        lower = torch.zeros(H, dtype=torch.float64)
        upper = torch.zeros(H, dtype=torch.float64)
        ops = []
        if rank > 0:
            ops += [dist.P2POp(dist.isend, own[:H].clone(), rank - 1), dist.P2POp(dist.irecv, lower, rank - 1)]
        if rank + 1 < WORLD:
            ops += [dist.P2POp(dist.isend, own[-H:].clone(), rank + 1), dist.P2POp(dist.irecv, upper, rank + 1)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        halo = np.concatenate([lower.numpy(), own.numpy(), upper.numpy()])
        # local rows of A p, columns shifted into the haloed index space
        q = np.empty(nloc)
        for i in range(lo, hi):
            acc = 0.0
            for k in range(a.rowptr[i], a.rowptr[i + 1]):
                acc = acc + a.vals[k] * halo[a.cols[k] - lo + H]
            q[i - lo] = acc
        # group partials of {q.p, q.q} at the local geometry, placed at the global group slots
        ngl = nloc // GS
        contrib = np.stack([q * p[lo:hi], q * q], axis=1)
        part_local = orc.stage1(contrib, ngl, GS)
        gathered = [torch.zeros_like(torch.from_numpy(part_local)) for _ in range(WORLD)]
        dist.all_gather(gathered, torch.from_numpy(part_local))
        full = np.concatenate([g.numpy() for g in gathered], axis=0)
        totals = orc.stage2(full)
        out[rank] = (q, full, totals)
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_and_partials_allgather_bitwise():
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(port, out), nprocs=WORLD, join=True)
    a, _ = orc.poisson3d(SIDE)
    n = SIDE ** 3
    p = np.random.default_rng(7).random(n)
    q_ref = orc.csr_spmv(a, p)
    contrib = np.stack([q_ref * p, q_ref * q_ref], axis=1)
    part_ref = orc.stage1(contrib, n // GS, GS)
    tot_ref = orc.stage2(part_ref)
    q_all = np.concatenate([out[r][0] for r in range(WORLD)])
    assert np.array_equal(q_all.view(np.uint64), q_ref.view(np.uint64))
    for r in range(WORLD):
        assert np.array_equal(out[r][1].view(np.uint64), part_ref.view(np.uint64))
        assert np.array_equal(np.asarray(out[r][2]).view(np.uint64), np.asarray(tot_ref).view(np.uint64))


def test_slab_geometry_rules():
    import paper_1410_4054_b200 as pk

    g = pk.slab_geometry(512, 65536)
    assert (g.n_groups, g.group_size) == (2048, 65536)  # C4: 256 groups per rank at 8 GPUs
    for world in (1, 2, 4, 8):
        nloc = 512 ** 3 // world
        assert nloc % 65536 == 0 and nloc >= 512 * 512
    with pytest.raises(ValueError):
        pk.slab_geometry(10, 64)

"""Multi-rank path on CPU (world_size 2 and 3, torch.distributed gloo): the library's partition /
exchange plan (ieti_plan_*, partition.cpp) reproduces the global jump operators.

Each rank keeps its local multiplier set (owned first, then ghosts) and exchanges with the plan's
lists exactly as the NCCL path does (forward: owner -> ghost copies before B^T / B_D^T; reverse:
ghost partial sums -> owner, added in ascending peer order after B / B_D).  The result on the
owned rows must equal the oracle's global B w and B_D w (readings R12),
and B^T / B_D^T of the local copies must equal the global products on every local patch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(P, send_lists, recv_lists, vals_send, nrecv):
    """one grouped exchange: per peer send vals_send[peer], receive nrecv[peer] doubles"""
    reqs, bufs = [], {}
    for i, q in enumerate(P["peers"]):
        if len(send_lists[i]):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(vals_send[i])), int(q)))
        if nrecv[i]:
            bufs[i] = torch.zeros(nrecv[i], dtype=torch.float64)
            reqs.append(dist.irecv(bufs[i], int(q)))
    for r in reqs:
        r.wait()
    return {i: b.numpy() for i, b in bufs.items()}


def _lists(P):
    sp, rp = P["send_ptr"], P["recv_ptr"]
    snd = [P["send_idx"][sp[i]:sp[i + 1]] for i in range(len(P["peers"]))]
    rcv = [P["recv_idx"][rp[i]:rp[i + 1]] for i in range(len(P["peers"]))]
    return snd, rcv


def halo_fwd(P, v):
    snd, rcv = _lists(P)
    got = _exchange(P, snd, rcv, [v[s] for s in snd], [len(r) for r in rcv])
    for i, r in enumerate(rcv):
        if len(r):
            v[r] = got[i]


def halo_rev(P, v):
    snd, rcv = _lists(P)
    got = _exchange(P, rcv, snd, [v[r] for r in rcv], [len(s) for s in snd])
    add = np.zeros(P["n_own"])
    for i in sorted(got):                       # ascending peer order, as k_rsum
        np.add.at(add, snd[i], got[i])
    v[:P["n_own"]] += add


def _worker(rank, world, port, case, owner_kind, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1705_04531_b200 as lib
        from oracle.topology import Topology
        from workloads import make_workload

        name, kw = case
        wl = make_workload(name, **kw)
        owner = None
        if owner_kind == "modulo":
            owner = [k % world for k in range(wl.n_patches)]
        P = lib.partition_plan(wl, rank, world, owner)
        T = Topology(wl.patches, wl.primal)
        loc = P["local_mult"].astype(np.int64)
        n_own = P["n_own"]
        lp = P["local_patches"]
        own_ref = np.array(owner) if owner is not None else np.repeat(np.arange(world), np.diff(
            [wl.n_patches * r // world for r in range(world + 1)]))
        assert list(lp) == [k for k in range(wl.n_patches) if own_ref[k] == rank]
        # owned multipliers = those whose k+ patch is local (R12 canonical rows)
        kplus = np.array([m[0] for m in T.mult])
        assert set(loc[:n_own]) == set(np.nonzero(own_ref[kplus] == rank)[0])
        rng = np.random.default_rng(0)
        lam = rng.standard_normal(T.n_lambda)
        w = [rng.standard_normal(T.B[k].shape[1]) for k in range(T.n_patches)]
        # forward halo: ghosts receive the owners' values
        v = np.full(len(loc), np.nan)
        v[:n_own] = lam[loc[:n_own]]
        halo_fwd(P, v)
        assert np.array_equal(v, lam[loc])
        # B^T, B_D^T of local patches need only the local set
        for k in lp:
            for op in (T.B, T.BD):
                Bk = op[k].tocsr()
                outside = np.setdiff1d(np.arange(T.n_lambda), loc)
                assert abs(Bk[outside]).sum() == 0.0
                np.testing.assert_allclose(Bk[loc].T @ v, Bk.T @ lam, rtol=0, atol=1e-14)
        # reverse: partial sums of B w, B_D w over local patches -> owners
        for op in (T.B, T.BD):
            part = sum((op[k] @ w[k] for k in lp), np.zeros(T.n_lambda))[loc].copy()
            halo_rev(P, part)
            ref = sum((op[k] @ w[k] for k in range(T.n_patches)), np.zeros(T.n_lambda))
            np.testing.assert_allclose(part[:n_own], ref[loc[:n_own]], rtol=0, atol=1e-13)
        # every global multiplier is owned by exactly one rank
        cnt = torch.zeros(T.n_lambda, dtype=torch.float64)
        cnt[torch.from_numpy(loc[:n_own])] = 1.0
        dist.all_reduce(cnt)
        assert torch.all(cnt == 1.0)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,case,owner_kind", [
    (2, ("C4", dict(m=4, grid=(2, 2, 2))), "blocks"),      # multiplicity-4 edges across the cut
    (2, ("C4", dict(m=4, grid=(2, 2, 2))), "modulo"),
    (3, ("C5", dict(m=4, grid=(3, 2, 2))), "blocks"),      # V+E+F, three ranks
    (2, ("C3", dict(m=8, grid=(4, 3))), "modulo"),         # 2D annulus, V+E
])
def test_exchange_plan_reproduces_global_jumps(world, case, owner_kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, owner_kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]


def test_default_partition_blocks():
    import paper_1705_04531_b200 as lib
    from workloads import make_workload
    wl = make_workload("C1")
    seen = []
    for r in range(3):
        P = lib.partition_plan(wl, r, 3)
        seen += list(P["local_patches"])
    assert seen == list(range(wl.n_patches))
    with pytest.raises(lib.IetiError):
        lib.partition_plan(wl, 0, 2, patch_owner=[0, 5, 1, 1])

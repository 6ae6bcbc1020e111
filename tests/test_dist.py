"""Multi-process (world_size 2, gloo, CPU) tests of the partitioning logic.

* instance sharding: the union of per-rank results equals the single-process
  batch (configs 1/2 shard with no data-path collective);
* row sharding: an MFZ trajectory integrated with the gram rows split across
  ranks and the contraction input all-gathered after every Euler step is
  bit-identical to the unsharded integration (config 4's exchange protocol),
  the per-rank step restating solver_mfz.cpp:47-88 with the oracle's
  canonical contraction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_00366_b200 import sharding


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _instance_worker(rank, world, port, q):
    from oracle import oracle as O
    _init(rank, world, port)
    insts = [O.gen_instance(48, 0.5 + 0.1 * (s % 3), 0.2, 0.01, s) for s in range(1, 6)]
    costs = [sharding.instance_cost(i.N, i.M, 200, 3) for i in insts]
    mine = sharding.instance_shard(costs, world, rank)
    hp = O.baseline_params(velo=2, n_steps=200)
    out = np.zeros((len(insts), 48))
    for b in mine:
        res = O.solve(insts[b], "mfz-bn", hp, seed=O.mix_seed(insts[b].seed, 1))
        out[b] = res["R"] * res["sigma"]
    t = torch.from_numpy(out)
    dist.all_reduce(t)  # disjoint blocks: the sum is the gather
    if rank == 0:
        q.put(t.numpy())
    dist.destroy_process_group()


def _row_worker(rank, world, port, q):
    from oracle import oracle as O
    _init(rank, world, port)
    N = 300
    inst = O.gen_instance(N, 0.6, 0.2, 0.01, 9)
    p = O.Problem(inst, O.CANON)
    G, hz, D = p.G, p.hz, p.gram_diag
    hp = O.baseline_params(n_steps=120)
    r0, r1 = sharding.row_shard(N, world, rank, quantum=64)
    Np = sharding.padded_rows(N, world, quantum=64)
    per = Np // world
    R = p.hz.copy()
    g = O.Rng(77)
    c = np.array([0.01 * g.gauss() for _ in range(N)])
    e = np.ones(N)
    rt = np.sqrt(hp.tau)
    pumps = O.pump_table(hp)
    eta = 0.5
    thresh = eta * eta / 4.0 * rt
    w = np.zeros(Np)
    w[:N] = R * (c > 0)
    for k in range(hp.n_steps):
        # local rows: h_i = (rt/2)(D_i w_i - G_i . w + hz_i), canonical order
        cl, el = c[r0:r1].copy(), e[r0:r1].copy()
        wn = np.zeros(per)
        for t_, i in enumerate(range(r0, r1)):
            gw = O.canon_dot(G[i], w[:N])
            h = (rt / 2.0) * ((D[i] * w[i] - gw) + hz[i])
            co, eo = O.mfz_step(cl[t_:t_ + 1], el[t_:t_ + 1], pumps[k], hp, eta,
                                R[i:i + 1], np.array([h]))
            cl[t_], el[t_] = co[0], eo[0]
            wn[t_] = R[i] * (1.0 if cl[t_] > 0 else 0.0)
        c[r0:r1], e[r0:r1] = cl, el
        # exchange: all-gather the w slices (and the state, for the check below)
        parts = [torch.zeros(per, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(wn))
        w = torch.cat(parts).numpy()
        cp = [torch.zeros(per, dtype=torch.float64) for _ in range(world)]
        cpad = np.zeros(per)
        cpad[: r1 - r0] = c[r0:r1]
        dist.all_gather(cp, torch.from_numpy(cpad))
        c = torch.cat(cp).numpy()[:N].copy()
    if rank == 0:
        ref = p.run_mfz(R, hp, eta, O.MFZ_BN, O.Rng(77))
        q.put((c, ref["c"]))
    dist.destroy_process_group()


def _spawn(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=fn, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    out = q.get(timeout=600)
    for p_ in ps:
        p_.join(timeout=600)
        assert p_.exitcode == 0
    return out


def test_instance_shard_plan():
    costs = [1.0] * 10
    parts = [sharding.instance_shard(costs, 4, r) for r in range(4)]
    assert [len(p) for p in parts] == [3, 2, 3, 2] or sum(len(p) for p in parts) == 10
    assert sorted(i for p in parts for i in p) == list(range(10))
    skew = [5.0, 1, 1, 1, 1, 1]
    a, b = (sharding.instance_shard(skew, 2, r) for r in range(2))
    assert list(a) == [0] and list(b) == [1, 2, 3, 4, 5]


def test_row_shard_plan():
    N, world = 1000, 4
    spans = [sharding.row_shard(N, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == N
    assert all(s[1] == t[0] for s, t in zip(spans, spans[1:]))
    assert sharding.padded_rows(N, world) % (world * 128) == 0


def test_instance_sharding_gloo(O):
    got = _spawn(_instance_worker)
    insts = [O.gen_instance(48, 0.5 + 0.1 * (s % 3), 0.2, 0.01, s) for s in range(1, 6)]
    hp = O.baseline_params(velo=2, n_steps=200)
    for b, inst in enumerate(insts):
        res = O.solve(inst, "mfz-bn", hp, seed=O.mix_seed(inst.seed, 1))
        assert np.array_equal(got[b], res["R"] * res["sigma"])


def test_row_sharded_step_gloo(O):
    c, ref = _spawn(_row_worker)
    assert np.array_equal(c, ref)

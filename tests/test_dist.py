"""Multi-process (world_size 2, gloo, CPU) tests of the partitioning logic.

* instance sharding: the union of per-rank results equals the single-process
  batch (configs 1/2 shard with no data-path collective);
* row sharding: an MFZ trajectory integrated with the gram rows split across
  ranks and the contraction input all-gathered after every Euler step is
  bit-identical to the unsharded integration (config 4's exchange protocol),
  the per-rank step restating solver_mfz.cpp:47-88 with the oracle's
  canonical contraction;
* tile sharding (config 4 on the symmetric path): the runtime's own super-row
  partition (cimcs_tile_shard) covers every upper-triangle tile exactly once,
  and the per-rank products of the owned tiles (G w and G^T w of each tile),
  all-reduced, give G w on every rank -- an MFZ trajectory integrated that
  way on two ranks matches the unsharded integration and is identical on
  both ranks (the replicated-state invariant).
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


def _tile_worker(rank, world, port, q):
    from oracle import oracle as O
    _init(rank, world, port)
    T = 16  # tile edge of this host restatement (the GPU uses 128)
    N = 150
    nRB = -(-N // T)
    inst = O.gen_instance(N, 0.6, 0.2, 0.01, 11)
    p = O.Problem(inst, O.EXPLICIT)
    G = np.zeros((nRB * T, nRB * T))
    G[:N, :N] = p.G
    P0, P1 = sharding.tile_shard(nRB, world, rank)
    S = 4
    mine = [(I, J) for P in range(P0, P1) for I in range(P * S, min(nRB, P * S + S))
            for J in range(I, nRB)]
    hp = O.baseline_params(velo=1, n_steps=60)
    rng = O.Rng(O.mix_seed(11, 1))
    c = np.array([rng.gauss() for _ in range(N)]) * 0.01
    e = np.ones(N)
    R = p.hz.copy()
    traj = []
    for k in range(hp.n_steps):
        w = np.zeros(nRB * T)
        w[:N] = R * (c > 0)
        part = np.zeros(nRB * T)
        for I, J in mine:  # each stored tile feeds both uses (sym_kernels.cuh)
            g = G[I * T:(I + 1) * T, J * T:(J + 1) * T]
            part[I * T:(I + 1) * T] += g @ w[J * T:(J + 1) * T]
            if I != J:
                part[J * T:(J + 1) * T] += g.T @ w[I * T:(I + 1) * T]
        t = torch.from_numpy(part)
        dist.all_reduce(t)  # one collective per step; every rank gets the same sum
        Gw = t.numpy()[:N]
        h = 0.5 * ((p.gram_diag * w[:N] - Gw) + p.hz)  # BN field, tau = 1
        p_k = O.pump_table(hp)[k]
        c, e = O.mfz_step(c, e, p_k, hp, 0.5, R, h)
        traj.append(c.copy())
    n_tiles = torch.tensor([len(mine)])
    dist.all_reduce(n_tiles)
    q.put((rank, np.array(traj), int(n_tiles), nRB))
    dist.destroy_process_group()


def _spawn_all(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=fn, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    outs = [q.get(timeout=600) for _ in ps]
    for p_ in ps:
        p_.join(timeout=600)
        assert p_.exitcode == 0
    return sorted(outs, key=lambda o: o[0])


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


def test_tile_shard_plan():
    """Contiguous super-rows, every rank non-empty, balanced by tile count."""
    for nRB, world in ((782, 8), (782, 2), (16, 2), (130, 4)):
        spans = [sharding.tile_shard(nRB, world, r) for r in range(world)]
        nSB = -(-nRB // 4)
        assert spans[0][0] == 0 and spans[-1][1] == nSB
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        tiles = []
        for P0, P1 in spans:
            tiles.append(sum(min(4, nRB - 4 * P) * (nRB - 4 * P) - (min(4, nRB - 4 * P) *
                             (min(4, nRB - 4 * P) - 1)) // 2 for P in range(P0, P1)))
        assert sum(tiles) == nRB * (nRB + 1) // 2
        if nRB >= 130:
            assert max(tiles) <= 1.35 * sum(tiles) / world, tiles


def test_tile_sharded_step_gloo(O):
    outs = _spawn_all(_tile_worker)
    (_, t0, n_tiles, nRB), (_, t1, _, _) = outs
    assert n_tiles == nRB * (nRB + 1) // 2  # every tile streamed by exactly one rank
    assert np.array_equal(t0, t1)            # replicated state stays identical
    # the unsharded integration with the dense product
    N = 150
    inst = O.gen_instance(N, 0.6, 0.2, 0.01, 11)
    p = O.Problem(inst, O.EXPLICIT)
    hp = O.baseline_params(velo=1, n_steps=60)
    rng = O.Rng(O.mix_seed(11, 1))
    c = np.array([rng.gauss() for _ in range(N)]) * 0.01
    e = np.ones(N)
    R = p.hz.copy()
    for k in range(hp.n_steps):
        w = R * (c > 0)
        h = 0.5 * ((p.gram_diag * w - p.G @ w) + p.hz)
        c, e = O.mfz_step(c, e, O.pump_table(hp)[k], hp, 0.5, R, h)
        assert np.allclose(t0[k], c, rtol=1e-9, atol=1e-12)

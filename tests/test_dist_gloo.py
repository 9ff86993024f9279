"""World-size-2 gloo tests of the multi-rank host logic on CPU (no GPU).

* shard table: gw_shard_rows / gw_check_shards from libgwdp.so (host-only entry points), the
  table exchanged with the same all-gather the host communicator uses;
* the host-callback communicator's marshalling (dist.host_comm + torch_allgather over gloo),
  invoked exactly as libgwdp.so invokes it;
* the exchange algebra of the sharded gradient: each rank forms its rows of
  G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y from its own rows of T plus the ranks' all-gathered
  column moments (sum_j T_jq, sum_j x_j T_jq) only, and must reproduce the oracle's full
  gradient rows.
"""

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2404_08970_b200 import dist as D
        ag = D.torch_allgather()
        res = {}
        # ---- shard table ----
        n = 1001
        r0, nl = D.shard_rows(n, world, rank)
        tab = np.frombuffer(ag(np.array([r0, nl], dtype=np.int64).tobytes()), dtype=np.int64).reshape(world, 2)
        D.check_shards(tab, n)
        res["tab"] = tab.tolist()
        # ---- the host communicator's callback, called the way libgwdp.so calls it ----
        comm = D.host_comm(world, rank, ag)
        payload = np.arange(5, dtype=np.float64) + 10.0 * rank
        recv = np.zeros(5 * world)
        rc = comm._keep(payload.ctypes.data_as(C.c_void_p), recv.ctypes.data_as(C.c_void_p), payload.nbytes, None)
        res["cb"] = (rc, recv.tolist())
        comm.close()
        # ---- sharded gradient algebra from gathered column moments ----
        rng = np.random.default_rng(3)
        N, M = 60, 47
        x, y = np.sort(rng.random(N)), np.sort(rng.random(M))
        p, qv = rng.dirichlet(np.ones(N)), rng.dirichlet(np.ones(M))
        T = rng.random((N, M)) / (N * M)
        a0, k = D.shard_rows(N, world, rank)
        Tl, xl = T[a0:a0 + k], x[a0:a0 + k]
        mom = np.concatenate([Tl.sum(0), xl @ Tl])  # this rank's column moments
        allm = np.frombuffer(ag(mom.tobytes()), dtype=np.float64).reshape(world, 2, M)
        DY = np.abs(y[:, None] - y[None, :])
        S_above = allm[:rank, 0].sum(0)
        X_above = allm[:rank, 1].sum(0)
        S_below = allm[rank + 1:, 0].sum(0)
        X_below = allm[rank + 1:, 1].sum(0)
        B = Tl @ DY
        V = (np.abs(xl[:, None] - xl[None, :]) @ B
             + xl[:, None] * (S_above @ DY)[None, :] - (X_above @ DY)[None, :]
             + (X_below @ DY)[None, :] - xl[:, None] * (S_below @ DY)[None, :])
        c, c2 = O.const_term(x, y, p, qv)
        Gl = 2.0 * (c[a0:a0 + k, None] + c2[None, :]) - 4.0 * V
        Go = O.grad_prescribed(x, y, p, qv, T)[a0:a0 + k]
        res["grad_err"] = float(np.max(np.abs(Gl - Go)) / np.max(np.abs(Go)))
        tdist.destroy_process_group()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_gloo_world2_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert isinstance(out[r], dict), out[r]
    assert out[0]["tab"] == [[0, 501], [501, 500]] == out[1]["tab"]
    for r in range(world):
        rc, recv = out[r]["cb"]
        assert rc == 0
        assert recv == [0.0, 1.0, 2.0, 3.0, 4.0, 10.0, 11.0, 12.0, 13.0, 14.0]
        assert out[r]["grad_err"] <= 1e-12


def test_shard_rows_and_check_shards_host_only():
    from paper_2404_08970_b200 import GwError
    from paper_2404_08970_b200 import dist as D
    for n, R in [(10, 3), (65536, 8), (7, 7), (5, 1)]:
        tab = [D.shard_rows(n, R, r) for r in range(R)]
        D.check_shards(tab, n)
        assert sum(t[1] for t in tab) == n and max(t[1] for t in tab) - min(t[1] for t in tab) <= 1
    with pytest.raises(GwError) as e:
        D.check_shards([(0, 5), (6, 4)], 10)
    assert e.value.code == "GW_ERR_DIM_MISMATCH"
    with pytest.raises(GwError):
        D.check_shards([(0, 5), (5, 4)], 10)

"""World-size-2 CPU tests (gloo) of the multi-GPU path's host logic.

The GPU ranks' compute is stood in for by the oracle's per-shard partials
(oracle.partials), exchanged with a real torch.distributed allreduce; this
checks the decomposition the NCCL path relies on ("dataset ...
divided among the number of threads" + merge + one master update):
  - contiguous shards cover [0, N) exactly once;
  - mu^0 assembled by an allreduce of owner-gathered rows (zeros elsewhere) is
    exactly x[init_idx];
  - the sum over ranks of shard partials equals the single-process step;
  - every rank computes bit-identical mu^{t+1} and E, so all stop together;
  - the NCCL unique id broadcast (paper_2405_12052_b200.dist) agrees on ranks.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2405_12052_b200 import datagen
        from paper_2405_12052_b200 import dist as kdist
        out = {}
        # unique id broadcast used by bench.py / init_comm
        uid = kdist.broadcast_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        out["uid_equal"] = all(i == ids[0] for i in ids) and len(uid) == 128

        w = datagen.WORKLOADS["NS"]
        N = 40_001
        a, b = kdist.shard(N, world, rank)
        Xs = datagen.generate(w, a, b - a, N=N)
        init = datagen.init_indices(w, N=N)
        K, d = w.K, w.d
        # CC1: owners contribute their rows, zeros elsewhere (k_init_gather + allreduce)
        mu = np.zeros((K, d))
        own = (init >= a) & (init < b)
        mu[own] = Xs[init[own] - a].astype(np.float64)
        t = torch.from_numpy(mu)
        dist.all_reduce(t)
        mu = t.numpy().copy()
        X = datagen.generate(w, N=N)
        out["mu0_exact"] = np.array_equal(mu, X[init].astype(np.float64))
        # a few distributed Lloyd iterations vs the single-process oracle
        Es, mus = [], []
        ok_step = True
        for it in range(4):
            p = oracle.partials(Xs, mu)
            vec = np.concatenate([p["sums"].ravel(), p["counts"].astype(np.float64), [p["J"]]])
            tv = torch.from_numpy(vec)
            dist.all_reduce(tv)   # CC2
            vec = tv.numpy()
            sums = vec[:K * d].reshape(K, d)
            counts = vec[K * d:K * d + K].astype(np.int64)
            J = vec[-1]
            o = oracle.step(X, mu)
            ok_step &= np.array_equal(counts, o["counts"])
            ok_step &= bool(np.all(np.abs(sums - o["sums"]) <= 1e-9 * np.abs(o["sums"]) + 1e-6))
            ok_step &= abs(J - o["J"]) <= 1e-9 * o["J"]
            mu_next, E = oracle.update(sums, counts, mu)
            Es.append(E)
            mus.append(mu_next.copy())
            mu = mu_next
        out["step_ok"] = bool(ok_step)
        # every rank must hold bit-identical centroids and E
        allmu = [None] * world
        dist.all_gather_object(allmu, (mus, Es))
        out["replicated"] = all(
            all(np.array_equal(x, y) for x, y in zip(m[0], allmu[0][0])) and m[1] == allmu[0][1]
            for m in allmu)
        out["shards"] = (a, b)
        # P2P exchange setup (kdist.enable_p2p): every rank maps the handles of
        # all ranks in rank order
        class FakeCtx:
            opened = None

            def p2p_handle(self):
                return bytes([rank + 1]) * 64

            def p2p_open(self, handles):
                self.opened = list(handles)
        fc = FakeCtx()
        on = kdist.enable_p2p(fc)
        out["p2p_handles_ok"] = on and fc.opened == [bytes([q + 1]) * 64 for q in range(world)]

        # all-or-nothing: if one rank cannot map its peers, every rank disables
        class FailingCtx(FakeCtx):
            disabled = False

            def p2p_open(self, handles):
                if rank == 1:
                    raise RuntimeError("no peer access")
                self.opened = list(handles)

            def p2p_disable(self):
                self.disabled = True
        fc2 = FailingCtx()
        on2 = kdist.enable_p2p(fc2)
        out["p2p_fallback_ok"] = (not on2) and (fc2.disabled == (rank != 1))
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the assertion below
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.parametrize("world", [2])
def test_distributed_decomposition_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r].get("error")
        assert res[r]["uid_equal"]
        assert res[r]["mu0_exact"]
        assert res[r]["step_ok"]
        assert res[r]["replicated"]
        assert res[r]["p2p_handles_ok"]
        assert res[r]["p2p_fallback_ok"]
    # shards cover [0, N) contiguously
    spans = sorted(res[r]["shards"] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == 40_001
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_shard_partition_properties():
    from paper_2405_12052_b200 import dist as kdist
    for N in [1, 5, 7, 100, 1_000_003]:
        for P in [1, 2, 3, 4, 8]:
            c = -(-N // P)
            if (P - 1) * c >= N:   # some rank would own no point: refused on every rank
                for r in range(P):
                    with pytest.raises(ValueError):
                        kdist.shard(N, P, r)
                continue
            spans = [kdist.shard(N, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
            sizes = [b - a for a, b in spans]
            c = -(-N // P)   # ceiling partition: full shards, then the remainder
            assert all(s == c for s in sizes[:N // c]) and sum(sizes) == N

"""The P2P exchange across PROCESSES on one GPU (the merge
over ranks of PAPER.md:97): two processes, each a rank of a P2P-only group
(opts.rank / opts.nranks, no NCCL), each maps the other's exchange buffer
with a real cudaIpcOpenMemHandle.  Ranks that spin on one another must not
run as separate launches on one GPU (B200_PROFILING.md), so the processes
take turns: while one runs kmeans_p2p_loopback -- every rank of the protocol
emulated in one cooperative launch over the REAL buffers, its own and the
peer process's -- the other waits on a pipe.  Each turn must produce the
rank-ordered sum bit for bit, which needs remote stores and loads through
the IPC mapping and system-scope flags to work in both directions.
"""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _rank(r, conn, q):
    sys.path.insert(0, ROOT)
    try:
        from paper_2405_12052_b200 import datagen
        from paper_2405_12052_b200 import kmeans as km
        w = datagen.WORKLOADS["C2"]
        N = 40_000
        a, b = datagen.shard_range(N, 2, r)
        X = datagen.generate(w, a, b - a, N=N)
        c = km.Context(X, w.K, device=0, rank=r, nranks=2, global_offset=a, global_N=N,
                       comm_timeout_s=10.0)
        conn.send(c.p2p_handle())
        handles = conn.recv()            # both ranks' handles, rank order
        c.p2p_open(handles)              # cudaIpcOpenMemHandle of the peer's buffer
        nE = w.K * w.d + w.K + 1
        out = {}
        for turn in range(2):
            msg = conn.recv()            # "go" for this rank's turn, "wait" otherwise
            if msg == ("go", r):
                rng = np.random.default_rng(100 * turn + r)
                vals = rng.standard_normal((3, 2, nE)) * 10.0 ** rng.integers(-3, 6, (3, 2, nE))
                got = c.p2p_loopback(vals)
                out[turn] = (vals, got)
            conn.send("done")
        info = c.info()
        c.close()
        q.put((r, {"out": out, "nranks": info["nranks"], "rank": info["rank"]}))
    except Exception:
        import traceback
        q.put((r, {"error": traceback.format_exc()}))


def test_p2p_exchange_across_processes_via_ipc():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pipes = [ctx.Pipe() for _ in range(2)]
    procs = [ctx.Process(target=_rank, args=(r, pipes[r][1], q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        parent = [pipes[r][0] for r in range(2)]
        handles = [parent[r].recv() for r in range(2)]
        assert all(len(h) == 64 for h in handles) and handles[0] != handles[1]
        for r in range(2):
            parent[r].send(handles)
        for turn in range(2):            # rank `turn` runs, the other waits
            for r in range(2):
                parent[r].send(("go", turn) if r == turn else ("wait", turn))
            # the idle rank answers at once; the active one after its launch
            for r in sorted(range(2), key=lambda r: r == turn):
                assert parent[r].recv() == "done"
        res = dict(q.get(timeout=300) for _ in range(2))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(2):
        assert "error" not in res[r], res[r].get("error")
        assert res[r]["nranks"] == 2 and res[r]["rank"] == r
    for turn in range(2):
        vals, got = res[turn]["out"][turn]
        for i in range(vals.shape[0]):
            expect = vals[i, 0] + vals[i, 1]   # rank order, fp64
            for r in range(2):
                assert np.array_equal(got[i, r], expect), (turn, i, r)

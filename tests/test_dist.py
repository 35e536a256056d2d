"""Multi-GPU path: 1-D destination partition + exchanges.

* CPU (`-m "not gpu"`): the host-side partition (gi_partition_ranges) against
  its definition, and a world_size-2 gloo run where each rank reduces its own
  share's in-degree histogram and both ranks must derive the same owner ranges.
* CPU: the host-staged collectives (paper_1805_00923_b200.hostcomm over gloo,
  world_size 2 and 3) against their definitions.
* GPU (`-m gpu`): P simulated ranks on ONE device (gi_local_group: one host
  thread per rank, collectives done by device copies) running the real
  partitioned build, PageRank and BFS; every rank's result is checked against
  the oracle on the whole graph.
* GPU, multi-process: world_size 2 and 3 gloo process groups, each process its
  own gi_context_create_hostcomm context on cuda:0 (the library's collectives
  staged through host memory into gloo), running the partitioned build from its
  own share of the edge list, PageRank (allgather and cross-process CUDA-IPC
  peer stores) and BFS end to end, checked against the oracle in every process.
"""
from __future__ import annotations

import os
import threading

import numpy as np
import pytest

import graphgen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gi():
    from paper_1805_00923_b200 import build

    build.build()
    from paper_1805_00923_b200 import gi as _gi

    return _gi


# ---------------------------------------------------------------- host logic (CPU)
def test_partition_ranges_definition(gi):
    rng = np.random.default_rng(3)
    for n, P in [(0, 1), (1, 4), (100, 3), (1000, 8), (4097, 2), (70000, 7)]:
        w = rng.integers(1, 50, n).astype(np.int64)
        if n > 10:
            w[:5] = 5000  # skew: hubs first
        pre = np.concatenate([[0], np.cumsum(w)])
        b = gi.gi_partition_ranges(n, P, pre)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        assert all(x % 32 == 0 for x in b[1:-1] if x != n)
        total = pre[-1]
        for r in range(1, P):
            if b[r] in (b[r - 1], n):
                continue
            # the cut is the first 32-aligned id at or after the equal-share point
            first = int(np.searchsorted(pre, total * r / P, side="left"))
            assert b[r] == min(max(-(-first // 32) * 32, b[r - 1]), n)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, ROOT)
    import graphgen as gg
    from paper_1805_00923_b200 import gi as g

    n = 1 << 12
    s, d = gg.rmat(12, 8, 0.57, 0.19, 0.19, 9)
    share = slice(rank, None, world)  # each rank holds an arbitrary share of the edges
    hist = torch.from_numpy(np.bincount(d[share][s[share] != d[share]], minlength=n).astype(np.int64))
    dist.all_reduce(hist)
    pre = np.concatenate([[0], np.cumsum(hist.numpy() + 1)])
    b = torch.from_numpy(g.gi_partition_ranges(n, world, pre))
    allb = [torch.zeros_like(b) for _ in range(world)]
    dist.all_gather(allb, b)
    q.put((rank, [x.tolist() for x in allb]))
    dist.destroy_process_group()


def test_gloo_two_ranks_agree_on_partition(gi):
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, allb in res:
        assert allb[0] == allb[1]  # both ranks computed identical owner ranges
        b = allb[0]
        assert b[0] == 0 and b[-1] == 1 << 12 and b[1] % 32 == 0


def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _spawn(target, world, *args, timeout=600):
    import multiprocessing as mp

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=timeout) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def _hostcomm_semantics_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, ROOT)
    from paper_1805_00923_b200.hostcomm import TorchDistComm

    c = TorchDistComm()
    out = {}
    for dt in (np.int32, np.int64, np.float64):
        a = (np.arange(5) * (rank + 1)).astype(dt)
        c.allreduce(a)
        out[np.dtype(dt).name] = a.tolist()
    # allgatherv: rank q owns bytes [off[q], off[q+1]) (uneven, one empty range)
    off = [0, 3, 3, 10][: world + 1] if world == 3 else [0, 7, 9]
    buf = np.zeros(off[-1], np.uint8)
    buf[off[rank]: off[rank + 1]] = 10 + rank
    c.allgatherv(buf, off)
    out["ag"] = buf.tolist()
    # alltoallv: rank r sends (r+1) * (q+1) bytes of value 16 r + q to rank q
    soff = [0]
    for qq in range(world):
        soff.append(soff[-1] + (rank + 1) * (qq + 1))
    send = np.concatenate([np.full((rank + 1) * (qq + 1), 16 * rank + qq, np.uint8) for qq in range(world)])
    roff = [0]
    for qq in range(world):
        roff.append(roff[-1] + (qq + 1) * (rank + 1))
    recv = np.zeros(roff[-1], np.uint8)
    c.alltoallv(send, soff, recv, roff)
    out["a2a"] = recv.tolist()
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_hostcomm_collectives_gloo(world):
    res = _spawn(_hostcomm_semantics_worker, world)
    tri = sum(range(1, world + 1))
    for rank, out in res:
        for name in ("int32", "int64", "float64"):
            assert out[name] == [i * tri for i in range(5)]
        off = [0, 3, 3, 10] if world == 3 else [0, 7, 9]
        want = []
        for qq in range(world):
            want += [10 + qq] * (off[qq + 1] - off[qq])
        assert out["ag"] == want
        want = []
        for qq in range(world):  # from rank qq: (qq+1)*(rank+1) bytes of 16 qq + rank
            want += [16 * qq + rank] * ((qq + 1) * (rank + 1))
        assert out["a2a"] == want


def _hostcomm_library_worker(rank, world, port, q, peer):
    import sys
    import traceback

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), GI_PR_PEER=peer, GI_BFS_PEER=peer)
    try:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, ROOT)
        import graphgen as gg
        import oracle as orc
        from paper_1805_00923_b200 import gi as G
        from paper_1805_00923_b200.hostcomm import TorchDistComm

        torch.cuda.set_device(0)
        ctx = G.Context(0, hostcomm=(rank, world, TorchDistComm()))
        bad = []
        for name, n, (s, d) in [("config1", gg.CONFIGS[1].n, gg.CONFIGS[1].edges()),
                                ("ragged", 30011, gg.random_digraph(30011, 250007, 6))]:
            go = orc.build_graph(n, s, d)
            sel = slice(rank, None, world)  # this process's share of the edge list
            g = G.Graph(ctx, n, s[sel].copy(), d[sel].copy())
            if g.m != go.m:
                bad.append((name, "m", g.m, go.m))
            for direction in (G.GI_PR_PULL, G.GI_PR_PULL_DIRECT, G.GI_PR_PUSH, G.GI_PR_PULL_BLOCKED):
                for dg in (0, 1):
                    got, st = g.pagerank(20, 0.85, direction=direction, dangling=dg, profile=True)
                    want = orc.pagerank(go, 20, 0.85, dg)
                    got = np.asarray(got, np.float64)
                    l1, rel = np.abs(got - want).sum(), (np.abs(got - want) / want).max()
                    if not (l1 <= 1e-5 and rel <= 1e-4):
                        bad.append((name, "pr", direction, dg, l1, rel))
                    if st.exchange != (2 if peer == "1" else 1):
                        bad.append((name, "exchange", st.exchange))
            for x in (0, n // 3, n - 1):
                depth = orc.bfs_depth(go, x)
                for pol in (G.GI_BFS_AUTO, G.GI_BFS_PUSH_ONLY, G.GI_BFS_PULL_ONLY):
                    par, st = g.bfs(x, policy=pol)
                    ok, msg = orc.validate_bfs(go, x, par, depth)
                    if not ok or st.edges_traversed != orc.reached_out_edges(go, depth):
                        bad.append((name, "bfs", x, pol, msg))
            pars, _ = g.bfs_multi([0, 1, 2, n - 1])
            for i, x in enumerate([0, 1, 2, n - 1]):
                ok, msg = orc.validate_bfs(go, x, pars[i])
                if not ok:
                    bad.append((name, "bfs_multi", x, msg))
            g.close()
        ctx.close()
        dist.destroy_process_group()
        q.put((rank, bad))
    except Exception:  # pragma: no cover - surfaced in the parent
        q.put((rank, [traceback.format_exc()]))


@pytest.mark.gpu
@pytest.mark.parametrize("peer", ["0", "1"])
@pytest.mark.parametrize("world", [2, 3])
def test_hostcomm_processes_end_to_end(world, peer):
    """world processes (gloo), each with its own hostcomm context on cuda:0: partitioned build
    from a per-process share of the edges, PageRank (peer=1: contrib stored into the other
    processes' replicas through CUDA IPC mappings) and BFS, all against the oracle."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("needs a CUDA device")
    res = _spawn(_hostcomm_library_worker, world, peer)
    for rank, bad in res:
        assert not bad, (rank, bad)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_wide_offsets(gi, P, monkeypatch):
    """The partitioned build, PR and BFS with int64 offsets (GI_OFFSETS64) on every rank."""
    test_partitioned_pagerank_and_bfs(gi, P, *CASES[1], "1", monkeypatch, wide=True)


# ---------------------------------------------------------------- simulated ranks on one GPU
def _run_ranks(gi, P, fn):
    """Run fn(rank, ctx) on P threads, each with its own local-group context."""
    grp = gi.gi_local_group_create(P)
    out, errs = [None] * P, []

    def body(r):
        try:
            ctx = gi.Context(0, local_group=grp, rank=r)
            try:
                out[r] = fn(r, ctx)
            finally:
                ctx.close()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    gi.gi_local_group_destroy(grp)
    assert not errs, errs
    return out


def _pr_ok(got, want):
    got = np.asarray(got, np.float64)
    l1 = np.abs(got - want).sum()
    rel = (np.abs(got - want) / want).max()
    assert l1 <= 1e-5 and rel <= 1e-4, (l1, rel)


CASES = [
    ("config1", graphgen.CONFIGS[1].n, lambda: graphgen.CONFIGS[1].edges()),
    ("random-ragged", 70001, lambda: graphgen.random_digraph(70001, 600007, 8)),
    ("instar-hub", 50001, lambda: graphgen.in_star(50000)),
    ("tiny", 37, lambda: graphgen.random_digraph(37, 120, 2)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("peer", ["1", "0"])
@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("name,n,make", CASES)
def test_partitioned_pagerank_and_bfs(gi, P, name, n, make, peer, monkeypatch, wide=False):
    """peer=1: the vertex update stores each owned row's contrib, and the BFS level
    kernels each owned next-frontier word, into every rank's replica (peer stores,
    SURVEY §8(f) NEXT #3); peer=0: the allgathers."""
    import torch

    monkeypatch.setenv("GI_PR_PEER", peer)
    monkeypatch.setenv("GI_BFS_PEER", peer)

    if not torch.cuda.is_available():
        pytest.fail("needs a CUDA device")
    s, d = make()
    go = oracle.build_graph(n, s, d)
    want = {dg: oracle.pagerank(go, 20, 0.85, dg) for dg in (0, 1)}
    srcs = [0, n // 3, n - 1]
    depth = {x: oracle.bfs_depth(go, x) for x in srcs}
    rng = np.random.default_rng(P)
    owner = rng.integers(0, P, len(s))  # arbitrary split of the edge list over ranks
    owner[: len(s) // 7] = 0  # uneven shares; some ranks may get almost nothing

    def fn(r, ctx):
        sel = owner == r
        g = gi.Graph(ctx, n, s[sel], d[sel], gi.GI_DEFAULT_FLAGS | (gi.GI_OFFSETS64 if wide else 0))
        res = {"m": g.m, "part": g.partition()}
        for direction in (gi.GI_PR_PULL, gi.GI_PR_PULL_DIRECT, gi.GI_PR_PUSH, gi.GI_PR_PULL_BLOCKED):
            for dg in (0, 1):
                res[("pr", direction, dg)] = g.pagerank(20, 0.85, direction=direction, dangling=dg)[0]
        res[("pr", "seg-small", 0)] = g.pagerank(20, 0.85, direction=gi.GI_PR_PULL_SEGMENTED, segment_size=1000)[0]
        for x in srcs:
            for pol in (gi.GI_BFS_AUTO, gi.GI_BFS_PUSH_ONLY, gi.GI_BFS_PULL_ONLY):
                res[("bfs", x, pol)] = g.bfs(x, policy=pol)
        g.close()
        return res

    out = _run_ranks(gi, P, fn)
    parts = sorted(o["part"] for o in out)
    assert parts[0][0] == 0 and parts[-1][1] == n
    assert all(parts[i][1] == parts[i + 1][0] for i in range(P - 1))
    assert sum(p[2] for p in parts) == go.m
    for o in out:
        assert o["m"] == go.m
        for key, val in o.items():
            if key[0] == "pr":
                _pr_ok(val, want[key[2]])
            elif key[0] == "bfs":
                par, st = val
                ok, msg = oracle.validate_bfs(go, key[1], par, depth[key[1]])
                assert ok, (name, P, key, msg)
                assert st.edges_traversed == oracle.reached_out_edges(go, depth[key[1]])

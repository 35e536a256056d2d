#!/usr/bin/env python3
"""Probe: can two processes on one GPU form an NCCL communicator through the library
(gi_context_create_dist) and run the partitioned PageRank / BFS? (diagnostics)

    python tools/nccl_same_gpu.py
"""
import multiprocessing as mp
import os
import socket
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, ROOT)
        import numpy as np
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        import graphgen as gg
        import oracle as orc
        from paper_1805_00923_b200 import gi as G

        torch.cuda.set_device(0)
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(G.gi_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ctx = G.Context(0, nccl=(rank, world, bytes(uid.numpy().tobytes())))
        cfg = gg.CONFIGS[1]
        s, d = cfg.edges()
        go = orc.build_graph(cfg.n, s, d)
        g = G.Graph(ctx, cfg.n, s[rank::world].copy(), d[rank::world].copy())
        got, st = g.pagerank(20, 0.85)
        want = orc.pagerank(go, 20, 0.85)
        l1 = float(np.abs(np.asarray(got, np.float64) - want).sum())
        par, bs = g.bfs(0)
        ok, msg = orc.validate_bfs(go, 0, par)
        g.close()
        ctx.close()
        q.put((rank, f"ok l1={l1:.2e} exchange={st.exchange} bfs={ok} {msg}"))
    except Exception:
        q.put((rank, traceback.format_exc()[-600:]))


if __name__ == "__main__":
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in ps:
        print(q.get(timeout=300))
    for p in ps:
        p.join(timeout=60)

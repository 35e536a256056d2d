"""Phase split of one bench e2e step (config 2 by default): graph create from pinned host edges (H2D inside),
first PageRank call (segmented layout build + calibration + 20 iterations, host output),
a second PageRank call, bfs_multi of the 64 sources into pinned host rows.

usage: python tools/e2e_split.py [CONFIG]
"""
import os
import resource
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1805_00923_b200 import gi  # noqa: E402

cfg = graphgen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
if cfg.scale >= 25:  # the bench's device generator (same edges as cfg.edges(), much faster)
    a_, b_, c_, _ = cfg.abcd
    ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a_, b_, c_, cfg.seed)
    s, d = ts.cpu().numpy(), td.cpu().numpy()
    del ts, td
    torch.cuda.empty_cache()
else:
    s, d = cfg.edges()
srcs = [int(x) for x in cfg.sources(s, d)]
flags = gi.GI_DEFAULT_FLAGS | (gi.GI_SYMMETRIZE if cfg.symmetrize else 0)
ctx = gi.Context(0)
hs, hd = torch.from_numpy(s).pin_memory(), torch.from_numpy(d).pin_memory()
hpr = torch.empty(cfg.n, dtype=torch.float32).pin_memory()
hbfs = torch.empty((len(srcs), cfg.n), dtype=torch.int32).pin_memory()
for rep in range(int(os.environ.get("E2E_REPS", "3"))):
    # wall time and this process's CPU time (user + system) per phase: a stall
    # with little CPU time is a wait (driver / DMA / scheduling), one with
    # system time is the kernel working for us (page faults, pinning)
    def now():
        o = os.times()
        r = resource.getrusage(resource.RUSAGE_SELF)
        return time.perf_counter(), o.user + o.system, r.ru_nvcsw, r.ru_majflt, r.ru_minflt

    t = [now()]
    g = gi.Graph(ctx, cfg.n, hs, hd, flags)
    torch.cuda.synchronize(); t.append(now())
    g.pagerank(cfg.pr_iters, cfg.damping, out=hpr)
    t.append(now())
    g.pagerank(cfg.pr_iters, cfg.damping, out=hpr)
    t.append(now())
    g.bfs_multi(srcs, out=hbfs)
    t.append(now())
    g.close()
    t.append(now())
    ms = [((b[0] - a[0]) * 1e3, (b[1] - a[1]) * 1e3) for a, b in zip(t, t[1:])]
    print("create %.1f/%.0f  pr#1 %.1f/%.0f  pr#2 %.1f/%.0f  bfs_multi(host) %.1f/%.0f  close %.1f/%.0f ms (wall/cpu)"
          % tuple(x for p in ms for x in p), flush=True)
    if os.environ.get("E2E_RUSAGE"):  # per phase: voluntary context switches, major / minor page faults
        print("   csw/majflt/minflt " + "  ".join("%d/%d/%d" % (b[2] - a[2], b[3] - a[3], b[4] - a[4])
                                                   for a, b in zip(t, t[1:])), flush=True)

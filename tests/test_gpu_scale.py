"""Oracle parity at the billion-edge configs on one B200 (BASELINE configs[3] and
configs[4]: RMAT s25 ef48, ~1.56 B directed edges, and RMAT s26 ef28
symmetrised, ~3.76 B directed edges, the only graph past 2^31 edges, so the
one that takes int64 offsets by size).

For each config, in the launch configuration bench.py times:

* PageRank, 20 iterations, d = 0.85 (auto pull kernel) element-wise against the
  full fp64 oracle: L1 <= 1e-5 and max per-vertex relative error <= 1e-4
  (north_star);
* BFS from the config's 16 seeded sources through gi_bfs_multi (the workload's
  call: one bit-parallel pass) AND through gi_bfs one source at a time, every
  parent vector validated against the oracle's depths (Graph500 rules: depths
  exact, tree edges exist), reached counts and TEPS edge counts (R16) equal.

The oracle (plain C, OpenMP) needs ~1 min (config 4) / ~3 min (config 5) of
the box's 16 host cores and ~100 GB of host RAM for config 5; the edge list
is generated on the device (the bit-exact twin of the host generator, checked
below) and copied to the host once.
"""
import os

import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu

PR_L1 = 1e-5
PR_REL = 1e-4


@pytest.fixture(scope="module")
def gi():
    from paper_1805_00923_b200 import build

    build.build()
    from paper_1805_00923_b200 import gi as _gi

    return _gi


def test_device_generator_matches_host():
    s, d = graphgen.rmat(20, 16, 0.57, 0.19, 0.19, 4, first=123456, count=100000)
    ts, td = graphgen.rmat_device(20, 16, 0.57, 0.19, 0.19, 4, first=123456, count=100000)
    assert np.array_equal(ts.cpu().numpy(), s) and np.array_equal(td.cpu().numpy(), d)


def _host_ram_gb():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
    except (ValueError, OSError):  # pragma: no cover
        return 0.0


@pytest.mark.slow
@pytest.mark.parametrize("cfg_idx", [4, 5])
def test_billion_edge_config_parity(gi, cfg_idx):
    import torch

    cfg = graphgen.CONFIGS[cfg_idx]
    need = {4: 60, 5: 120}[cfg_idx]
    if _host_ram_gb() < need:
        pytest.fail(f"config {cfg_idx} parity needs ~{need} GB of host RAM for the oracle "
                    f"({_host_ram_gb():.0f} GB here)")
    a, b, c, _ = cfg.abcd
    ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
    s, d = ts.cpu().numpy(), td.cpu().numpy()
    n = cfg.n
    ctx = gi.Context(0, torch.cuda.current_stream().cuda_stream)
    flags = gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE | (gi.GI_SYMMETRIZE if cfg.symmetrize else 0)
    g = gi.Graph(ctx, n, ts, td, flags)
    del ts, td
    torch.cuda.empty_cache()
    go = oracle.build_graph(n, s, d, symmetrize=cfg.symmetrize)
    sources = [int(x) for x in cfg.sources(s, d)]
    del s, d
    assert len(sources) == cfg.bfs_sources == 16
    assert g.m == go.m
    if cfg_idx == 5:
        assert g.m >= 2**31  # int64 offsets by size

    # ---- PageRank (the bench's call: auto pull kernel, 20 iterations)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    _, st = g.pagerank(cfg.pr_iters, cfg.damping, out=out)
    assert st.bytes_alg_per_iter == 4 * g.m + ((8 if g.m >= 2**31 else 4) + 12) * n
    # the auto pull kernel: segmented on the skewed config 4, propagation-blocked on config 5
    assert st.kernel == (gi.GI_PR_PULL_BLOCKED if cfg_idx == 5 else gi.GI_PR_PULL_SEGMENTED)
    got = out.cpu().numpy().astype(np.float64)
    want = oracle.pagerank(go, cfg.pr_iters, cfg.damping)
    l1 = np.abs(got - want).sum()
    rel = (np.abs(got - want) / want).max()
    assert l1 <= PR_L1 and rel <= PR_REL, f"{cfg.name}: L1={l1:.3e} maxrel={rel:.3e}"
    del got, want, out

    # ---- BFS: the workload's 16-source call (one bit-parallel pass) and per-source gi_bfs
    multi = torch.empty((len(sources), n), dtype=torch.int32, device="cuda")
    _, mst = g.bfs_multi(sources, out=multi)
    par = torch.empty(n, dtype=torch.int32, device="cuda")
    for i, src in enumerate(sources):
        depth = oracle.bfs_depth_levels(go, src)
        reached = int((depth >= 0).sum())
        tep = oracle.reached_out_edges(go, depth)
        ok, msg = oracle.validate_bfs(go, src, multi[i].cpu().numpy(), depth)
        assert ok, f"{cfg.name} gi_bfs_multi row {i} (src {src}): {msg}"
        assert mst[i].reached == reached and mst[i].edges_traversed == tep
        _, bs = g.bfs(src, out=par)
        ok, msg = oracle.validate_bfs(go, src, par.cpu().numpy(), depth)
        assert ok, f"{cfg.name} gi_bfs src {src}: {msg}"
        assert bs.reached == reached and bs.edges_traversed == tep
    g.close()
    ctx.close()

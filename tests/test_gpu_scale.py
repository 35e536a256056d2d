"""Billion-edge scale on one B200: BASELINE configs[3] (RMAT s25 ef48, ~1.5 B
directed edges after cleanup) end to end, checked by properties that hold at
any size (the fp64 oracle would need minutes and ~30 GB here):

* PageRank: mass conserved under the uniform rule (sum r = 1), r >= (1-d)/n,
  and the Jacobi relation between consecutive iterates recomputed one by one
  for sampled vertices from the raw edge list (torch on the device, fp64):
  r_20[v] = (1-d)/n + d * (sum_{u in in(v)} r_19[u]/outdeg(u) + D_19/n);
* BFS: Graph500 validation on the whole edge list — parent[s] = s, every tree
  edge exists, depth(parent) = depth - 1, every edge (u, v) with u reached has
  v reached and depth(v) <= depth(u) + 1 — plus edges_traversed.
The device generator is checked bit-for-bit against the host generator.
"""
import numpy as np
import pytest

import graphgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gi():
    from paper_1805_00923_b200 import build

    build.build()
    from paper_1805_00923_b200 import gi as _gi

    return _gi


def test_device_generator_matches_host():
    import torch

    s, d = graphgen.rmat(20, 16, 0.57, 0.19, 0.19, 4, first=123456, count=100000)
    ts, td = graphgen.rmat_device(20, 16, 0.57, 0.19, 0.19, 4, first=123456, count=100000)
    assert np.array_equal(ts.cpu().numpy(), s) and np.array_equal(td.cpu().numpy(), d)
    del torch


def _clean_edges(ts, td):
    keep = ts != td
    return ts[keep], td[keep]


@pytest.mark.slow
def test_config4_full_scale(gi):
    import torch

    cfg = graphgen.CONFIGS[4]
    a, b, c, _ = cfg.abcd
    ts, td = graphgen.rmat_device(cfg.scale, cfg.edge_factor, a, b, c, cfg.seed)
    n = cfg.n
    ctx = gi.Context(0, torch.cuda.current_stream().cuda_stream)
    g = gi.Graph(ctx, n, ts, td, gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
    assert g.m > 1_400_000_000
    outdeg = g.out_degrees(torch.empty(n, dtype=torch.int32, device="cuda")).to(torch.float64)
    assert int(outdeg.sum().item()) == g.m

    # ---- PageRank
    r20 = torch.empty(n, dtype=torch.float32, device="cuda")
    r19 = torch.empty(n, dtype=torch.float32, device="cuda")
    _, st = g.pagerank(20, cfg.damping, out=r20)
    g.pagerank(19, cfg.damping, out=r19)
    assert st.kernel == gi.GI_PR_PULL_SEGMENTED
    r20d, r19d = r20.double(), r19.double()
    assert abs(r20d.sum().item() - 1.0) < 1e-4
    assert r20d.min().item() >= (1 - cfg.damping) / n * (1 - 1e-4)
    dang = outdeg == 0
    D19 = r19d[dang].sum().item()
    u_all, v_all = _clean_edges(ts, td)
    rng = np.random.default_rng(4)
    # samples: the top hubs (internal hot rows) and random vertices with in-edges
    indeg_est = torch.bincount(v_all, minlength=n)
    hubs = torch.topk(indeg_est, 3).indices.cpu().numpy()
    cand = torch.nonzero(indeg_est > 0).flatten().cpu().numpy()
    samples = list(hubs) + list(rng.choice(cand, 5, replace=False))
    for v in samples:
        srcs = torch.unique(u_all[v_all == int(v)])  # dedup: one edge per (u, v)
        s = (r19d[srcs.long()] / outdeg[srcs.long()]).sum().item()
        want = (1 - cfg.damping) / n + cfg.damping * (s + D19 / n)
        got = r20d[int(v)].item()
        assert abs(got - want) <= 1e-4 * want, (int(v), got, want)

    # ---- BFS (Graph500-style validation on all edges)
    srcs_pick = torch.nonzero(outdeg > 0).flatten()[:: max(1, n // 7)][:2].cpu().numpy()
    for s0 in srcs_pick:
        par = torch.empty(n, dtype=torch.int32, device="cuda")
        _, bs = g.bfs(int(s0), out=par)
        p = par.long()
        assert p[int(s0)].item() == int(s0)
        reached = p >= 0
        # depth by pointer jumping over the parent tree
        # walk from every reached vertex itself, so depth(s) = 0 and depth(child of s) = 1
        steps = torch.zeros_like(p)
        cur = torch.where(reached, torch.arange(n, device=p.device), torch.full_like(p, int(s0)))
        for _ in range(64):
            moving = cur != int(s0)
            if not bool(moving.any()):
                break
            steps += moving.long()
            cur = torch.where(moving, p[cur], cur)
        assert not bool((cur != int(s0)).any()), "parent pointers do not reach the source"
        depth = torch.where(reached, steps, torch.full_like(p, -1))
        # tree edges exist: (parent[v], v) among the input pairs, checked by sorted-key membership
        key = torch.unique(u_all.long() * n + v_all.long())
        vv = torch.nonzero(reached).flatten()
        vv = vv[vv != int(s0)]
        tk = p[vv] * n + vv
        pos = torch.searchsorted(key, tk)
        assert bool((key[pos.clamp(max=len(key) - 1)] == tk).all()), "a tree edge is not in the graph"
        assert bool((depth[p[vv]] == depth[vv] - 1).all())
        # BFS optimality over all edges
        du, dv = depth[u_all.long()], depth[v_all.long()]
        ru = du >= 0
        assert bool((dv[ru] >= 0).all()) and bool((dv[ru] <= du[ru] + 1).all())
        assert bs.reached == int(reached.sum().item())
        assert bs.edges_traversed == int(outdeg[reached].sum().item())
    g.close()
    ctx.close()

"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * build: CSR bit-exact (integer work), degrees bit-exact;
  * PageRank (fp32 on the GPU vs fp64 oracle, same iteration count):
      L1 distance <= 1e-5 and max per-vertex relative error <= 1e-4;
  * BFS: depths bit-exact (derived from the parent tree by the validator),
    parent trees VALIDATED (several are correct, R8), never compared.
"""
from __future__ import annotations

import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu

PR_L1 = 1e-5
PR_REL = 1e-4


class _WideOffsets:
    """The binding with every graph built with GI_OFFSETS64: int64 CSR/CSC offsets, the layout
    of graphs past 2^31 edges (config 5), so the whole suite also runs the
    int64-offset kernel instantiations."""

    def __init__(self, mod):
        self._mod = mod

        class Graph(mod.Graph):
            def __init__(self, ctx, n, src, dst, flags=mod.GI_DEFAULT_FLAGS):
                super().__init__(ctx, n, src, dst, flags | mod.GI_OFFSETS64)

        self.Graph = Graph
        self.wide = True

    def __getattr__(self, k):
        return getattr(self._mod, k)


@pytest.fixture(scope="module", params=["off32", "off64"])
def gi(request):
    from paper_1805_00923_b200 import build

    build.build()
    from paper_1805_00923_b200 import gi as _gi

    return _WideOffsets(_gi) if request.param == "off64" else _gi


@pytest.fixture(scope="module")
def ctx(gi):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (there is no CPU fallback)")
    c = gi.Context(0)
    yield c
    c.close()


def _pr_check(got, want, what=""):
    got = np.asarray(got, np.float64)
    l1 = np.abs(got - want).sum()
    rel = (np.abs(got - want) / np.maximum(np.abs(want), 1e-300)).max() if len(want) else 0.0
    assert l1 <= PR_L1 and rel <= PR_REL, f"{what}: L1={l1:.3e} maxrel={rel:.3e}"
    return l1, rel


def _bfs_check(g_or, source, parent, what=""):
    depth = oracle.bfs_depth(g_or, source)
    ok, msg = oracle.validate_bfs(g_or, source, parent, depth)
    assert ok, f"{what}: {msg}"


FLAG_SETS = [
    ("default", None, dict(remove_self_loops=True, dedup=True, symmetrize=False)),
    ("no-relabel", "norelabel", dict(remove_self_loops=True, dedup=True, symmetrize=False)),
    ("sym", "sym", dict(remove_self_loops=True, dedup=True, symmetrize=True)),
    ("raw", "raw", dict(remove_self_loops=False, dedup=False, symmetrize=False)),
]


def _flags(gi, kind):
    f = gi.GI_REMOVE_SELF_LOOPS | gi.GI_DEDUP
    if kind == "norelabel":
        f |= gi.GI_NO_RELABEL
    elif kind == "sym":
        f |= gi.GI_SYMMETRIZE
    elif kind == "raw":
        f = 0
    return f


# ---------------------------------------------------------------- build (a1, a2)
@pytest.mark.parametrize("name,kind,oflags", FLAG_SETS)
def test_build_csr_bit_exact(gi, ctx, name, kind, oflags):
    for seed in range(3):
        n = [1, 37, 5000][seed]
        s, d = graphgen.random_digraph(n, 8 * n + 3, 100 + seed)
        g = gi.Graph(ctx, n, s, d, _flags(gi, kind))
        go = oracle.build_graph(n, s, d, **oflags)
        assert g.n == n and g.m == go.m
        off, idx = g.csr()
        assert np.array_equal(off, go.csr_off), name
        if kind == "raw":  # duplicates kept: compare as sorted multisets per row (order of equal keys)
            assert np.array_equal(idx, go.csr_idx)
        else:
            assert np.array_equal(idx, go.csr_idx), name
        assert np.array_equal(g.out_degrees(), go.outdeg.astype(np.int32))
        assert np.array_equal(g.in_degrees(), go.indeg.astype(np.int32))


def test_build_rmat_config1_bit_exact(gi, ctx):
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    go = oracle.build_graph(cfg.n, s, d)
    assert g.m == go.m
    off, idx = g.csr()
    assert np.array_equal(off, go.csr_off) and np.array_equal(idx, go.csr_idx)
    # edge-list checksum of the cleaned graph agrees on both sides
    src_o = np.repeat(np.arange(cfg.n, dtype=np.int32), np.diff(go.csr_off))
    src_g = np.repeat(np.arange(cfg.n, dtype=np.int32), np.diff(off))
    assert graphgen.edge_checksum(src_o, go.csr_idx) == graphgen.edge_checksum(src_g, idx)


@pytest.mark.parametrize("name,kind,oflags", [fs for fs in FLAG_SETS if fs[1] != "sym"])
def test_build_host_edges_pipelined(gi, ctx, name, kind, oflags):
    """gi_graph_create from host edges of >= 2^24 entries takes the pipelined build (H2D in chunks
    overlapped with the degree count, per-chunk key sorts, merge-path rounds): bit-exact CSR against
    the oracle and the device-edge build, PageRank on it against the oracle; an endpoint outside
    [0, n) in any chunk is an error."""
    import torch

    n = 1 << 20
    s, d = graphgen.rmat(20, 24, 0.57, 0.19, 0.19, 777)  # 25 M entries with self-loops and duplicates
    assert len(s) >= 1 << 24
    flags = _flags(gi, kind)
    g = gi.Graph(ctx, n, s, d, flags)
    go = oracle.build_graph(n, s, d, **oflags)
    assert g.m == go.m
    off, idx = g.csr()
    assert np.array_equal(off, go.csr_off) and np.array_equal(idx, go.csr_idx)
    assert np.array_equal(g.out_degrees(), go.outdeg.astype(np.int32))
    gd = gi.Graph(ctx, n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), flags | gi.GI_EDGES_ON_DEVICE)
    offd, idxd = gd.csr()
    assert np.array_equal(offd, off) and np.array_equal(idxd, idx)
    assert np.array_equal(gd.out_degrees(), g.out_degrees())
    gd.close()
    if kind != "raw":
        ph, _ = g.pagerank(5, 0.85)
        _pr_check(ph, oracle.pagerank(go, 5, 0.85), f"host-edge build {name}")
    g.close()
    for arr, pos, val in ((d, len(d) - 1, n), (s, len(s) // 3, -1), (d, 5, n + 7)):
        bad = arr.copy()
        bad[pos] = val
        args = (s, bad) if arr is d else (bad, d)
        with pytest.raises(gi.GiError) as e:
            gi.Graph(ctx, n, *args, flags)
        assert e.value.status == gi.GI_ERR_VERTEX_OUT_OF_RANGE


def test_build_device_edges_and_errors(gi, ctx):
    import torch

    s, d = graphgen.random_digraph(100, 1000, 5)
    ts, td = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
    g = gi.Graph(ctx, 100, ts, td, gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
    go = oracle.build_graph(100, s, d)
    off, idx = g.csr()
    assert np.array_equal(off, go.csr_off) and np.array_equal(idx, go.csr_idx)
    with pytest.raises(gi.GiError) as e:
        gi.Graph(ctx, 10, np.array([0, 10], np.int32), np.array([1, 1], np.int32))
    assert e.value.status == gi.GI_ERR_VERTEX_OUT_OF_RANGE
    with pytest.raises(gi.GiError) as e:
        gi.Graph(ctx, 10, np.array([0, -1], np.int32), np.array([1, 1], np.int32))
    assert e.value.status == gi.GI_ERR_VERTEX_OUT_OF_RANGE
    with pytest.raises(gi.GiError) as e:
        gi.Graph(ctx, 10, s[:0], d[:0], 1 << 20)
    assert e.value.status == gi.GI_ERR_INVALID_ARGUMENT
    with pytest.raises(gi.GiError) as e:
        gi.Graph(ctx, 10, s[:5], d[:5], gi.GI_EDGES_ON_DEVICE)  # host arrays flagged as device
    assert e.value.status == gi.GI_ERR_INVALID_ARGUMENT


# ---------------------------------------------------------------- PageRank (a3-a5)
PR_DIRS = ["pull", "push", "direct", "segmented", "partitioned", "blocked"]


def _dir(gi, name):
    return {"pull": gi.GI_PR_PULL, "push": gi.GI_PR_PUSH, "direct": gi.GI_PR_PULL_DIRECT,
            "segmented": gi.GI_PR_PULL_SEGMENTED, "partitioned": gi.GI_PR_PULL_PARTITIONED,
            "blocked": gi.GI_PR_PULL_BLOCKED}[name]


@pytest.mark.parametrize("direction", PR_DIRS)
def test_pr_small_families(gi, ctx, direction):
    cases = [
        ("cycle7", 7, *graphgen.cycle(7)),
        ("star", 51, *graphgen.star_bidirectional(50)),
        ("instar", 21, *graphgen.in_star(20)),
        ("K9", 9, *graphgen.complete(9)),
        ("path", 10, *graphgen.path(10)),
        ("empty", 5, np.zeros(0, np.int32), np.zeros(0, np.int32)),
        ("single", 1, np.zeros(0, np.int32), np.zeros(0, np.int32)),
    ]
    for name, n, s, d in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        for dangling in (gi.GI_DANGLING_UNIFORM, gi.GI_DANGLING_DROP):
            for iters in (0, 1, 2, 20):
                got, _ = g.pagerank(iters, 0.85, direction=_dir(gi, direction), dangling=dangling)
                want = oracle.pagerank(go, iters, 0.85, dangling)
                _pr_check(got, want, f"{name} it={iters} dangling={dangling}")


@pytest.mark.parametrize("direction", PR_DIRS)
def test_pr_exhaustive_tiny(gi, ctx, direction):
    # every digraph on 3 vertices, a sample on 4
    for n, masks in [(3, range(64)), (4, range(0, 4096, 37))]:
        pairs = [(u, v) for u in range(n) for v in range(n) if u != v]
        for mask in masks:
            s = np.array([u for i, (u, v) in enumerate(pairs) if mask >> i & 1], np.int32)
            d = np.array([v for i, (u, v) in enumerate(pairs) if mask >> i & 1], np.int32)
            g = gi.Graph(ctx, n, s, d)
            got, _ = g.pagerank(20, 0.85, direction=_dir(gi, direction))
            _pr_check(got, oracle.pagerank(oracle.build_graph(n, s, d), 20, 0.85), f"n={n} mask={mask}")


@pytest.mark.parametrize("direction", PR_DIRS)
@pytest.mark.parametrize("n,m0,seed", [(100, 50, 1), (1000, 20000, 2), (3000, 3000, 3), (20000, 200000, 4),
                                       (70001, 1000003, 5)])
def test_pr_random_ragged(gi, ctx, direction, n, m0, seed):
    """Sizes spanning several merge-path tiles with ragged tails and many dangling/isolated vertices."""
    s, d = graphgen.random_digraph(n, m0, seed)
    g = gi.Graph(ctx, n, s, d)
    go = oracle.build_graph(n, s, d)
    got, _ = g.pagerank(20, 0.85, direction=_dir(gi, direction))
    _pr_check(got, oracle.pagerank(go, 20, 0.85), f"n={n}")


@pytest.mark.parametrize("direction", PR_DIRS)
def test_pr_hub_rows_split_across_tiles(gi, ctx, direction):
    """In-star with 100k leaves: the centre's CSC row spans ~50 tiles (last-arriver fix-up)."""
    L = 100_000
    s, d = graphgen.in_star(L)
    s2, d2 = graphgen.star_bidirectional(L)
    for name, (ss, dd) in {"instar": (s, d), "bistar": (s2, d2)}.items():
        g = gi.Graph(ctx, L + 1, ss, dd)
        go = oracle.build_graph(L + 1, ss, dd)
        for dangling in (0, 1):
            got, _ = g.pagerank(20, 0.85, direction=_dir(gi, direction), dangling=dangling)
            _pr_check(got, oracle.pagerank(go, 20, 0.85, dangling), name)


@pytest.mark.parametrize("direction", PR_DIRS)
@pytest.mark.parametrize("relabel", [True, False])
def test_pr_config1(gi, ctx, direction, relabel):
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    flags = gi.GI_DEFAULT_FLAGS | (0 if relabel else gi.GI_NO_RELABEL)
    g = gi.Graph(ctx, cfg.n, s, d, flags)
    go = oracle.build_graph(cfg.n, s, d)
    got, st = g.pagerank(cfg.pr_iters, cfg.damping, direction=_dir(gi, direction))
    want = oracle.pagerank(go, cfg.pr_iters, cfg.damping)
    _pr_check(got, want, "config1")
    assert st.edge_launches == cfg.pr_iters


@pytest.mark.parametrize("seg,dblk", [(32, 0), (1000, 777), (4096, 50000), (20000, 0), (0, 3000)])
def test_pr_segmented_many_segments(gi, ctx, seg, dblk):
    """Small segment sizes and destination blocks: many (block, segment) units,
    pieces split across chunks and CTAs, tiny units gathered without staging."""
    cases = [(graphgen.CONFIGS[1].n, *graphgen.CONFIGS[1].edges()),
             (70001, *graphgen.random_digraph(70001, 1000003, 5)),
             (100001, *graphgen.in_star(100000)),
             (100001, *graphgen.star_bidirectional(100000))]
    for n, s, d in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        for dangling in (0, 1):
            got, st = g.pagerank(20, 0.85, direction=gi.GI_PR_PULL_SEGMENTED, dangling=dangling, segment_size=seg,
                                 dst_block=dblk)
            assert st.kernel == gi.GI_PR_PULL_SEGMENTED
            _pr_check(got, oracle.pagerank(go, 20, 0.85, dangling), f"seg={seg} dblk={dblk} n={n}")


@pytest.mark.parametrize("steal", ["0", "2"])
def test_pr_segmented_work_stealing(gi, ctx, steal, monkeypatch):
    """The segmented pull with CTAs stealing halves of each other's record ranges (forced on
    config 2's layout, ~1150 records per CTA, by GI_SEG_STEAL=2) and without (0): PR (repeated:
    every launch steals differently) and CC against the oracle."""
    monkeypatch.setenv("GI_SEG_STEAL", steal)
    cfg = graphgen.CONFIGS[2]
    s, d = cfg.edges()
    go = oracle.build_graph(cfg.n, s, d)
    want = oracle.pagerank(go, 20, 0.85)
    import torch

    ts, td = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
    for seg in (0, 20000):
        g = gi.Graph(ctx, cfg.n, ts, td, gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
        out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
        for _ in range(3):
            _, st = g.pagerank(20, 0.85, out=out, direction=gi.GI_PR_PULL_SEGMENTED, segment_size=seg)
            _pr_check(out.cpu().numpy(), want, f"steal={steal} seg={seg}")
        if seg == 0:
            lab = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
            g.cc(out=lab)
            assert (lab.cpu().numpy() == oracle.cc_labels(go)).all()
        g.close()


@pytest.mark.parametrize("z", [1, 1000, 4096, 30000, 0])
def test_pr_partitioned_many_partitions(gi, ctx, z):
    """Cache partitioning: the CSC split by source range
    into 2^k-vertex partitions (up to 32), one merge-path pass per partition;
    rows empty in a partition, hubs split across tiles, a single partition (z=0)."""
    cases = [(graphgen.CONFIGS[1].n, *graphgen.CONFIGS[1].edges()),
             (70001, *graphgen.random_digraph(70001, 1000003, 5)),
             (100001, *graphgen.in_star(100000)),
             (100001, *graphgen.star_bidirectional(100000)),
             (5, np.zeros(0, np.int32), np.zeros(0, np.int32))]
    for n, s, d in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        for dangling in (0, 1):
            got, st = g.pagerank(20, 0.85, direction=gi.GI_PR_PULL_PARTITIONED, dangling=dangling, segment_size=z)
            if go.m > 0:
                assert st.kernel == gi.GI_PR_PULL_PARTITIONED
            _pr_check(got, oracle.pagerank(go, 20, 0.85, dangling), f"z={z} n={n}")


def test_pr_blocked_hub_blocks_and_chunks(gi, ctx):
    """The propagation-blocked pull where its layout has many source chunks (n > 49152 per
    chunk), row blocks cut by edge count (a 200k-in-edge hub row, a 30k-leaf in-star) and
    sparse tiles: against the oracle under both dangling rules."""
    n = 150_001
    s0, d0 = graphgen.random_digraph(n, 400_000, 21)
    hub_src = np.arange(1, 200_001, dtype=np.int32) % n
    s = np.concatenate([s0, hub_src, np.arange(30_000, dtype=np.int32) + 100_000])
    d = np.concatenate([d0, np.zeros(len(hub_src), np.int32), np.full(30_000, 99_999, np.int32)])
    go = oracle.build_graph(n, s, d)
    g = gi.Graph(ctx, n, s, d)
    for dg in (0, 1):
        got, st = g.pagerank(20, 0.85, direction=gi.GI_PR_PULL_BLOCKED, dangling=dg)
        assert st.kernel == gi.GI_PR_PULL_BLOCKED
        _pr_check(got, oracle.pagerank(go, 20, 0.85, dg), f"blocked dangling={dg}")
    g.close()


def test_pr_device_output_and_damping_edges(gi, ctx):
    import torch

    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    go = oracle.build_graph(cfg.n, s, d)
    out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
    g.pagerank(20, 0.85, out=out)
    _pr_check(out.cpu().numpy(), oracle.pagerank(go, 20, 0.85), "device out")
    for damp in (0.0, 1.0, 0.5):
        got, _ = g.pagerank(7, damp)
        _pr_check(got, oracle.pagerank(go, 7, damp), f"damping {damp}")
    for bad in (-0.1, 1.1, float("nan")):
        with pytest.raises(gi.GiError):
            g.pagerank(3, bad)
    with pytest.raises(gi.GiError):
        g.pagerank(-1, 0.85)


def test_pr_stress_repeat(gi, ctx):
    """100 repetitions of both directions stay within tolerance (missing atomics would not)."""
    s, d = graphgen.rmat(12, 16, 0.57, 0.19, 0.19, 21)
    n = 1 << 12
    g = gi.Graph(ctx, n, s, d)
    want = oracle.pagerank(oracle.build_graph(n, s, d), 20, 0.85)
    for rep in range(50):
        for direction in PR_DIRS:
            got, _ = g.pagerank(20, 0.85, direction=_dir(gi, direction))
            _pr_check(got, want, f"rep {rep} {direction}")


# ---------------------------------------------------------------- BFS (a6-a9)
POLICIES = ["auto", "push", "pull"]


def _pol(gi, p):
    return {"auto": gi.GI_BFS_AUTO, "push": gi.GI_BFS_PUSH_ONLY, "pull": gi.GI_BFS_PULL_ONLY}[p]


@pytest.mark.parametrize("policy", POLICIES)
def test_bfs_small_families(gi, ctx, policy):
    import json
    import os

    gd = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bfs_path4.json")))
    g = gi.Graph(ctx, gd["n"], np.array(gd["src"], np.int32), np.array(gd["dst"], np.int32))
    par, _ = g.bfs(gd["source"], policy=_pol(gi, policy))
    assert par.tolist() == gd["parent"]  # unique tree: compared exactly
    cases = [
        ("star", 31, *graphgen.star_bidirectional(30), [0, 5]),
        ("K8", 8, *graphgen.complete(8), [0, 7]),
        ("reverse", 2, np.array([1], np.int32), np.array([0], np.int32), [0, 1]),
        ("disconnected", 6, np.array([0, 1, 3], np.int32), np.array([1, 0, 4], np.int32), [0, 3, 5]),
        ("single", 1, np.zeros(0, np.int32), np.zeros(0, np.int32), [0]),
        ("cycle", 100, *graphgen.cycle(100), [0, 99]),
    ]
    for name, n, s, d, sources in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        for src in sources:
            par, st = g.bfs(src, policy=_pol(gi, policy))
            _bfs_check(go, src, par, f"{name} src={src}")


@pytest.mark.parametrize("policy", POLICIES)
def test_bfs_random_and_grid(gi, ctx, policy):
    for n, m0, seed in [(50, 200, 1), (4097, 30000, 2), (30000, 90000, 3)]:
        s, d = graphgen.random_digraph(n, m0, seed)
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        for src in (0, n // 2, n - 1):
            par, st = g.bfs(src, policy=_pol(gi, policy))
            _bfs_check(go, src, par, f"rand n={n} src={src}")
    R, C = 97, 61
    s, d = graphgen.grid(R, C, 0.1, 3)
    g = gi.Graph(ctx, R * C, s, d)
    go = oracle.build_graph(R * C, s, d)
    par, st = g.bfs(0, policy=_pol(gi, policy))
    _bfs_check(go, 0, par, "grid")
    s, d = graphgen.grid(40, 30, 0.0, 3)
    g = gi.Graph(ctx, 1200, s, d)
    par, st = g.bfs(0, policy=_pol(gi, policy))
    # undropped grid: depth(r, c) = r + c; reconstruct depth from the tree
    depth = np.full(1200, -1)
    depth[0] = 0
    for _ in range(100):
        upd = (depth < 0) & (par >= 0)
        depth[upd] = np.where(depth[par[upd]] >= 0, depth[par[upd]] + 1, -1)
    rr, cc = np.divmod(np.arange(1200), 30)
    assert np.array_equal(depth, rr + cc)
    assert st.levels == 40 + 30 - 1


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("relabel", [True, False])
def test_bfs_config1(gi, ctx, policy, relabel):
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    flags = gi.GI_DEFAULT_FLAGS | (0 if relabel else gi.GI_NO_RELABEL)
    g = gi.Graph(ctx, cfg.n, s, d, flags)
    go = oracle.build_graph(cfg.n, s, d)
    sources = [0] + graphgen.pick_sources(cfg.n, s, d, 8, 1001).tolist()
    for src in sources:
        par, st = g.bfs(src, policy=_pol(gi, policy))
        depth = oracle.bfs_depth(go, src)
        ok, msg = oracle.validate_bfs(go, src, par, depth)
        assert ok, f"src={src}: {msg}"
        assert st.reached == int((depth >= 0).sum())
        assert st.edges_traversed == oracle.reached_out_edges(go, depth)
        assert st.levels == depth.max() + 1
        if policy == "push":
            assert st.pull_levels == 0
    # the direction-optimising run actually switched direction on this graph
    _, st = g.bfs(0, policy=gi.GI_BFS_AUTO)
    assert 0 < st.pull_levels < st.levels


@pytest.mark.parametrize("batch", ["per_source", "bitparallel"])
@pytest.mark.parametrize("where", ["host", "device"])
def test_bfs_multi(gi, ctx, where, batch):
    """gi_bfs_multi == k gi_bfs runs (valid trees, same depths and stats):
    config 1 and a high-diameter grid (per-source: sources rerun through the
    small-grid handover), per-source and bit-parallel batches."""
    bmode = {"per_source": gi.GI_BFS_BATCH_PER_SOURCE, "bitparallel": gi.GI_BFS_BATCH_BITPARALLEL}[batch]
    import torch

    cfg = graphgen.CONFIGS[1]
    s1, d1 = cfg.edges()
    s3, d3 = graphgen.grid(64, 64, 0.1, 3)
    cases = [(cfg.n, s1, d1, [0] + graphgen.pick_sources(cfg.n, s1, d1, 9, 1001).tolist()),
             (64 * 64, s3, d3, [0, 4095, 2080, 0])]
    for n, s, d, sources in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        out = (torch.full((len(sources), n), 7, dtype=torch.int32, device="cuda") if where == "device"
               else np.full((len(sources), n), 7, np.int32))
        par, stats = g.bfs_multi(sources, out=out, batch=bmode)
        par = par.cpu().numpy() if where == "device" else par
        for i, src in enumerate(sources):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"n={n} src={src}: {msg}"
            _, one = g.bfs(src)
            assert (stats[i].levels, stats[i].reached, stats[i].edges_traversed) == \
                (one.levels, one.reached, one.edges_traversed)
    g = gi.Graph(ctx, 10, *graphgen.cycle(10))
    with pytest.raises(gi.GiError) as e:
        g.bfs_multi([0, 10], batch=bmode)
    assert e.value.status == gi.GI_ERR_VERTEX_OUT_OF_RANGE
    out, st = g.bfs_multi([], batch=bmode)
    assert out.shape == (0, 10) and st == []


def test_bfs_multi_bitparallel_batches(gi, ctx):
    """More than 64 sources (two bit-parallel passes), repeated sources, every
    direction policy; each row validated against the oracle."""
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    go = oracle.build_graph(cfg.n, s, d)
    sources = graphgen.pick_sources(cfg.n, s, d, 70, 77).tolist() + [0, 0]
    for policy in POLICIES:
        par, stats = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, policy=_pol(gi, policy))
        for i, src in enumerate(sources):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"{policy} src={src}: {msg}"
            assert stats[i].reached == int((depth >= 0).sum())
            assert stats[i].edges_traversed == oracle.reached_out_edges(go, depth)
            assert stats[i].levels == depth.max() + 1


@pytest.mark.parametrize("k", [8, 16, 17, 32, 33, 64])
def test_bfs_multi_bitparallel_mask_widths(gi, ctx, k):
    """The pull levels gather frontier masks narrowed to 16 bits (k <= 16) or 32 bits (k <= 32),
    else the 64-bit masks: every width at its boundary, every direction policy."""
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    go = oracle.build_graph(cfg.n, s, d)
    sources = graphgen.pick_sources(cfg.n, s, d, k, 100 + k).tolist()
    for policy in POLICIES:
        par, st = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, policy=_pol(gi, policy))
        for i, src in enumerate(sources):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"k={k} {policy} src={src}: {msg}"
            assert st[i].reached == int((depth >= 0).sum())
    g.close()


@pytest.mark.parametrize("k", [8, 16, 17, 32, 33, 64])
def test_bfs_multi_segmented_or_pull(gi, ctx, k):
    """Bit-parallel pull levels as an OR pass over the segmented layout (GI_MS_PULL_SEGMENTED):
    every width it takes (16-bit parent-scan masks for k <= 16, 32-bit up to 32, two 32-bit OR
    passes and 64-bit parent scans above), every direction
    policy, on layouts with one, two and many source segments / destination blocks (pieces split
    across records and CTAs, unstaged sparse units), a hub row of 100k in-edges (a heavy row
    resolved by a warp) and a graph without relabelling.
    Each row is validated against the oracle (exact depths, valid parents); the stats say which
    kernel ran."""
    cfg = graphgen.CONFIGS[1]
    cases = [("rmat", cfg.n, *cfg.edges(), 0, 0),
             ("rmat-small-segments", cfg.n, *cfg.edges(), 4096, 20000),
             ("random", 70001, *graphgen.random_digraph(70001, 1000003, 5), 1000, 0),
             ("star", 100001, *graphgen.star_bidirectional(100000), 0, 0)]
    for name, n, s, d, seg, dblk in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        if seg or dblk:  # the layout PageRank builds with these parameters, reused by the BFS
            g.pagerank(1, 0.85, direction=gi.GI_PR_PULL_SEGMENTED, segment_size=seg, dst_block=dblk)
        sources = graphgen.pick_sources(n, s, d, k, 300 + k).tolist() if name != "star" else \
            list(range(1, k)) + [0]
        for policy in POLICIES:
            par, st = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, policy=_pol(gi, policy),
                                  pull_kernel=gi.GI_MS_PULL_SEGMENTED)
            assert st[0].pull_or_levels == st[0].pull_levels
            if policy == "pull":
                assert st[0].pull_or_levels > 0
            for i, src in enumerate(sources):
                depth = oracle.bfs_depth(go, src)
                ok, msg = oracle.validate_bfs(go, src, par[i], depth)
                assert ok, f"{name} k={k} {policy} src={src}: {msg}"
                assert st[i].reached == int((depth >= 0).sum())
                assert st[i].levels == depth.max() + 1
                assert st[i].edges_traversed == oracle.reached_out_edges(go, depth)
        g.close()
    # no relabelling (internal ids = input ids, no permutation in the parent scans)
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d, gi.GI_DEFAULT_FLAGS | gi.GI_NO_RELABEL)
    go = oracle.build_graph(cfg.n, s, d)
    sources = graphgen.pick_sources(cfg.n, s, d, k, 400 + k).tolist()
    par, st = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, policy=gi.GI_BFS_PULL_ONLY,
                          pull_kernel=gi.GI_MS_PULL_SEGMENTED)
    assert st[0].pull_or_levels == st[0].pull_levels > 0
    for i, src in enumerate(sources):
        ok, msg = oracle.validate_bfs(go, src, par[i], oracle.bfs_depth(go, src))
        assert ok, f"norelabel k={k} src={src}: {msg}"
    g.close()


def test_bfs_multi_or_pull_auto(gi, ctx):
    """AUTO pull kernel: after a PageRank call has built the segmented layout, the dense pull
    levels of a 16-source pass run as OR passes (rows missing sources hold > m/4 in-edges);
    GI_MS_PULL_ROWS keeps the row pull. Both validated against the oracle."""
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    go = oracle.build_graph(cfg.n, s, d)
    sources = graphgen.pick_sources(cfg.n, s, d, 16, 501).tolist()
    _, st0 = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL)
    assert st0[0].pull_or_levels == 0  # no layout yet
    g.pagerank(2, 0.85, direction=gi.GI_PR_PULL_SEGMENTED)
    for pk in (gi.GI_MS_PULL_AUTO, gi.GI_MS_PULL_ROWS):
        par, st = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, pull_kernel=pk)
        assert (st[0].pull_or_levels > 0) == (pk == gi.GI_MS_PULL_AUTO and st[0].pull_levels > 0)
        for i, src in enumerate(sources):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"pull_kernel={pk} src={src}: {msg}"
            assert st[i].edges_traversed == st0[i].edges_traversed
    # pull-only: the late levels pull only the listed rows still missing a source; ROWS pulls every row
    for pk in (gi.GI_MS_PULL_AUTO, gi.GI_MS_PULL_ROWS):
        par, st = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, policy=gi.GI_BFS_PULL_ONLY,
                              pull_kernel=pk)
        assert (st[0].pull_sparse_levels > 0) == (pk == gi.GI_MS_PULL_AUTO)
        for i, src in enumerate(sources):
            ok, msg = oracle.validate_bfs(go, src, par[i], oracle.bfs_depth(go, src))
            assert ok, f"pull-only pull_kernel={pk} src={src}: {msg}"
    with pytest.raises(gi.GiError) as e:
        g.bfs_multi(sources, pull_kernel=3)
    assert e.value.status == gi.GI_ERR_INVALID_ARGUMENT
    g.close()


@pytest.mark.parametrize("k", [16, 33, 64])
def test_bfs_multi_listed_row_pull(gi, ctx, k):
    """Late pull levels over the listed rows still missing a source (the rows' in-edges < m/64),
    every mask width (16-bit gathers, 32/64-bit masks): a symmetrised RMAT graph under the pull-only
    policy, where the rows of the giant component complete and the last levels turn sparse.
    Validated against the oracle."""
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d, gi.GI_DEFAULT_FLAGS | gi.GI_SYMMETRIZE)
    go = oracle.build_graph(cfg.n, s, d, symmetrize=True)
    sources = graphgen.pick_sources(cfg.n, s, d, k, 600 + k).tolist()
    for pk in (gi.GI_MS_PULL_AUTO, gi.GI_MS_PULL_SEGMENTED):
        par, st = g.bfs_multi(sources, batch=gi.GI_BFS_BATCH_BITPARALLEL, policy=gi.GI_BFS_PULL_ONLY,
                              pull_kernel=pk)
        if pk == gi.GI_MS_PULL_AUTO:  # no layout: row pulls, the late ones listed
            assert st[0].pull_sparse_levels > 0
        else:  # forced OR passes at every pull level (the layout built on demand)
            assert st[0].pull_or_levels == st[0].pull_levels
        for i, src in enumerate(sources):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"k={k} pull_kernel={pk} src={src}: {msg}"
            assert st[i].reached == int((depth >= 0).sum())
    g.close()


def test_bfs_multi_bitparallel_edge_cases(gi, ctx):
    """Bit-parallel passes on degenerate inputs: no edges; isolated and sink
    sources; k = 1, 64 and 65; a 100k-leaf star under every direction policy —
    pull-only makes the hub's 100k in-edges a split heavy row whose chunks race
    on the same bits."""
    bp = gi.GI_BFS_BATCH_BITPARALLEL
    # no edges: every row holds only its own source
    g = gi.Graph(ctx, 100, np.zeros(0, np.int32), np.zeros(0, np.int32))
    srcs = [3, 7, 7, 99, 0, 50, 51, 52, 53, 54]
    par, st = g.bfs_multi(srcs, batch=bp)
    for i, s in enumerate(srcs):
        want = np.full(100, -1, np.int32)
        want[s] = s
        assert (par[i] == want).all()
        assert (st[i].reached, st[i].levels, st[i].edges_traversed) == (1, 1, 0)
    # RMAT: isolated vertices and sinks as sources, k = 1 / 64 / 65
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    go = oracle.build_graph(cfg.n, s, d)
    outdeg = np.bincount(s[s != d], minlength=cfg.n)
    indeg = np.bincount(d[s != d], minlength=cfg.n)
    isolated = np.nonzero((outdeg == 0) & (indeg == 0))[0][:3].tolist()
    sinks = np.nonzero((outdeg == 0) & (indeg > 0))[0][:3].tolist()
    live = graphgen.pick_sources(cfg.n, s, d, 70, 5).tolist()
    for srcs in ([live[0]], isolated + sinks + live[:58], live[:65]):
        par, st = g.bfs_multi(srcs, batch=bp)
        for i, src in enumerate(srcs):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"k={len(srcs)} src={src}: {msg}"
            assert st[i].reached == int((depth >= 0).sum())
            assert st[i].levels == depth.max() + 1
    # 100k-leaf bidirectional star, sources = 64 leaves (+ the hub)
    L = 100_000
    s, d = graphgen.star_bidirectional(L)
    g = gi.Graph(ctx, L + 1, s, d)
    go = oracle.build_graph(L + 1, s, d)
    srcs = list(range(1, 64)) + [0]
    for policy in POLICIES:
        par, st = g.bfs_multi(srcs, batch=bp, policy=_pol(gi, policy))
        for i, src in enumerate(srcs):
            depth = oracle.bfs_depth(go, src)
            ok, msg = oracle.validate_bfs(go, src, par[i], depth)
            assert ok, f"star {policy} src={src}: {msg}"


def test_bfs_stress_repeat(gi, ctx):
    s, d = graphgen.rmat(13, 16, 0.57, 0.19, 0.19, 33)
    n = 1 << 13
    g = gi.Graph(ctx, n, s, d)
    go = oracle.build_graph(n, s, d)
    depth = oracle.bfs_depth(go, 0)
    for rep in range(40):
        for policy in POLICIES:
            par, _ = g.bfs(0, policy=_pol(gi, policy))
            ok, msg = oracle.validate_bfs(go, 0, par, depth)
            assert ok, f"rep {rep} {policy}: {msg}"


def test_bfs_errors_and_device_output(gi, ctx):
    import torch

    s, d = graphgen.cycle(10)
    g = gi.Graph(ctx, 10, s, d)
    with pytest.raises(gi.GiError) as e:
        g.bfs(10)
    assert e.value.status == gi.GI_ERR_VERTEX_OUT_OF_RANGE
    with pytest.raises(gi.GiError):
        g.bfs(-1)
    out = torch.empty(10, dtype=torch.int32, device="cuda")
    g.bfs(3, out=out)
    assert out.cpu().tolist() == [9, 0, 1, 3, 3, 4, 5, 6, 7, 8]


def test_offsets_width_takes_effect(gi, ctx):
    """B_alg = 4m + (o+12)n reports the offset width o the graph was built with."""
    s, d = graphgen.CONFIGS[1].edges()
    n = graphgen.CONFIGS[1].n
    g = gi.Graph(ctx, n, s, d)
    _, st = g.pagerank(2, 0.85)
    o = 8 if getattr(gi, "wide", False) else 4
    assert st.bytes_alg_per_iter == 4 * g.m + (o + 12) * n
    g.close()


# ---------------------------------------------------------------- full-size configs (BASELINE configs[1], [2])
@pytest.fixture(scope="module")
def full_graphs():
    """Oracle graphs of configs 2 and 3 (built once; ~1 min of host time each)."""
    return {}


@pytest.mark.parametrize("cfg_idx", [2, 3])
def test_full_config_parity(gi, ctx, full_graphs, cfg_idx):
    """The bench workload at full size, in the launch configuration bench.py times:
    PageRank (auto pull kernel) against the full fp64 oracle, and BFS from
    several sources validated against oracle depths."""
    cfg = graphgen.CONFIGS[cfg_idx]
    s, d = cfg.edges()
    go = oracle.build_graph(cfg.n, s, d)
    import torch

    g = gi.Graph(ctx, cfg.n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(),
                 gi.GI_DEFAULT_FLAGS | gi.GI_EDGES_ON_DEVICE)
    assert g.m == go.m
    out = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
    _, st = g.pagerank(cfg.pr_iters, cfg.damping, out=out)
    want = oracle.pagerank(go, cfg.pr_iters, cfg.damping)
    got = out.cpu().numpy()
    _pr_check(got, want, cfg.name)
    assert abs(got.astype(np.float64).sum() - 1.0) < 1e-5  # mass conserved (uniform rule)
    sources = cfg.sources(s, d).tolist() if cfg.source_seed else [0]
    # the bench's exact call: every source of the workload (64 on config 2) in one gi_bfs_multi
    # (AUTO: one bit-parallel pass of 64 sources), all rows validated
    allp = torch.empty((len(sources), cfg.n), dtype=torch.int32, device="cuda")
    _, ast = g.bfs_multi(sources, out=allp)
    few = sources[:4]
    par = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    multi = torch.empty((len(few), cfg.n), dtype=torch.int32, device="cuda")
    bitp = torch.empty((len(few), cfg.n), dtype=torch.int32, device="cuda")
    _, mst = g.bfs_multi(few, out=multi, batch=gi.GI_BFS_BATCH_PER_SOURCE)
    _, bst = g.bfs_multi(few, out=bitp, batch=gi.GI_BFS_BATCH_BITPARALLEL)
    for i, src in enumerate(sources):
        depth = oracle.bfs_depth_levels(go, int(src))
        runs = [("gi_bfs_multi (bench call)", allp[i], ast[i])]
        if i < len(few):
            _, bs = g.bfs(int(src), out=par)
            runs += [("gi_bfs", par, bs), ("gi_bfs_multi per-source", multi[i], mst[i]),
                     ("gi_bfs_multi bit-parallel", bitp[i], bst[i])]
        for what, p, st in runs:
            ok, msg = oracle.validate_bfs(go, int(src), p.cpu().numpy(), depth)
            assert ok, f"{cfg.name} {what} src={src}: {msg}"
            assert st.edges_traversed == oracle.reached_out_edges(go, depth)
            assert st.reached == int((depth >= 0).sum())


# ---------------------------------------------------------------- PageRankDelta
PRD_POLICIES = ["auto", "push", "pull"]


def _prd_pol(gi, p):
    return {"auto": gi.GI_PRD_AUTO, "push": gi.GI_PRD_PUSH_ONLY, "pull": gi.GI_PRD_PULL_ONLY}[p]


@pytest.mark.parametrize("policy", PRD_POLICIES)
def test_prdelta_parity(gi, ctx, policy):
    """GPU PageRankDelta vs the fp64 oracle on the same rounds. The frontier test
    |Delta| > eps*Rank is taken in fp64 on both sides (the paper's precision);
    the per-round frontier sizes must agree exactly, ranks within the PR bars."""
    cases = [("config1", graphgen.CONFIGS[1].n, *graphgen.CONFIGS[1].edges()),
             ("random", 20000, *graphgen.random_digraph(20000, 200000, 4)),
             ("bistar", 5001, *graphgen.star_bidirectional(5000))]
    for name, n, s, d in cases:
        g = gi.Graph(ctx, n, s, d)
        go = oracle.build_graph(n, s, d)
        for eps, iters in [(0.0, 10), (0.1, 10), (0.01, 15)]:
            want, fs = oracle.pagerank_delta(go, iters, 0.85, eps, return_frontiers=True)
            got, st = g.pagerank_delta(iters, 0.85, eps, policy=_prd_pol(gi, policy))
            assert st.active_total == int(fs.sum()), (name, eps, st.active_total, fs.tolist())
            got = np.asarray(got, np.float64)
            l1 = np.abs(got - want).sum()
            rel = (np.abs(got - want) / np.maximum(want, 1e-300)).max()
            assert l1 <= 1e-5 and rel <= 1e-4, (name, eps, policy, l1, rel)
        if policy == "auto" and name == "config1":
            # the paper's point: the frontier shrinks, so later rounds switch to push
            _, st = g.pagerank_delta(15, 0.85, 0.01)
            assert st.rounds >= 3 and 0 < st.pull_rounds < st.rounds


def test_prdelta_equals_pagerank_drop_at_eps0(gi, ctx):
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    want = oracle.pagerank(oracle.build_graph(cfg.n, s, d), 12, 0.85, oracle.DROP)
    got, _ = g.pagerank_delta(12, 0.85, 0.0)
    _pr_check(got, want, "prdelta eps=0 vs PR drop")


# ---------------------------------------------------------------- connected components (NEXT #4)
def _cc_cases():
    cfg = graphgen.CONFIGS[1]
    s1, d1 = cfg.edges()
    sr, dr = graphgen.rmat(18, 8, 0.57, 0.19, 0.19, 21)
    s3, d3 = graphgen.grid(128, 128, 0.3, 5)  # dropped edges split the grid into pieces
    ps = np.arange(999, dtype=np.int32)
    return [
        ("config1", cfg.n, s1, d1, False),
        ("config1-sym", cfg.n, s1, d1, True),
        ("rmat18-sym", 1 << 18, sr, dr, True),
        ("grid128", 128 * 128, s3, d3, False),
        ("path", 1000, ps, ps + 1, False),
        ("path-reversed", 1000, ps + 1, ps, False),
        ("star", 100_001, *graphgen.star_bidirectional(100_000), False),
        ("edgeless", 17, np.zeros(0, np.int32), np.zeros(0, np.int32), False),
    ]


@pytest.mark.parametrize("policy", POLICIES)
def test_cc_parity(gi, ctx, policy):
    """gi_cc == the oracle's fixed point (min input id over ancestors), exactly,
    on directed and symmetrised RMAT, a fragmented grid, paths, a 100k-leaf star
    and an edgeless graph, under every direction policy."""
    for name, n, s, d, sym in _cc_cases():
        flags = gi.GI_DEFAULT_FLAGS | (gi.GI_SYMMETRIZE if sym else 0)
        g = gi.Graph(ctx, n, s, d, flags)
        go = oracle.build_graph(n, s, d, symmetrize=sym)
        want = oracle.cc_labels(go)
        got, st = g.cc(policy=_pol(gi, policy))
        assert (got == want).all(), f"{name} {policy}: {int((got != want).sum())} labels differ"
        assert st.rounds >= 1 or n == 0
        g.close()


def test_cc_device_output_and_errors(gi, ctx):
    import torch

    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d, gi.GI_DEFAULT_FLAGS | gi.GI_SYMMETRIZE)
    want = oracle.cc_labels(oracle.build_graph(cfg.n, s, d, symmetrize=True))
    out = torch.full((cfg.n,), -7, dtype=torch.int32, device="cuda")
    got, st = g.cc(out=out, profile=True)
    assert (got.cpu().numpy() == want).all()
    assert st.total_ms > 0 and st.launches >= 2
    # repeated calls reuse the state
    got2, _ = g.cc()
    assert (got2 == want).all()
    with pytest.raises(gi.GiError) as e:
        g.cc(policy=7)
    assert e.value.status == gi.GI_ERR_INVALID_ARGUMENT


# ---------------------------------------------------------------- SSSP (NEXT #4)
@pytest.mark.parametrize("policy", POLICIES)
def test_sssp_parity(gi, ctx, policy):
    """gi_sssp == Dijkstra on the oracle's graph with graphgen's weights (exact
    integers): directed and symmetrised RMAT, a fragmented grid, a path, a 100k-leaf
    star; every direction policy; several sources and weight seeds."""
    cfg = graphgen.CONFIGS[1]
    s1, d1 = cfg.edges()
    s3, d3 = graphgen.grid(96, 96, 0.2, 7)
    ps = np.arange(499, dtype=np.int32)
    cases = [("config1", cfg.n, s1, d1, False, [0, 5, 777]),
             ("config1-sym", cfg.n, s1, d1, True, [3]),
             ("grid96", 96 * 96, s3, d3, False, [0, 4000]),
             ("path", 500, ps, ps + 1, False, [0, 250, 499]),
             ("star", 100_001, *graphgen.star_bidirectional(100_000), False, [0, 77])]
    for name, n, s, d, sym, srcs in cases:
        flags = gi.GI_DEFAULT_FLAGS | (gi.GI_SYMMETRIZE if sym else 0)
        g = gi.Graph(ctx, n, s, d, flags)
        go = oracle.build_graph(n, s, d, symmetrize=sym)
        for seed in (1, 99):
            w = oracle.csr_weights(go, seed)
            for src in srcs:
                want = oracle.sssp(go, src, w)
                got, st = g.sssp(src, seed=seed, policy=_pol(gi, policy))
                assert (got.astype(np.int64) == want).all(), \
                    f"{name} seed={seed} src={src} {policy}: {int((got != want).sum())} distances differ"
        g.close()


@pytest.mark.parametrize("policy", POLICIES)
def test_sssp_weighted_parity(gi, ctx, policy):
    """gi_sssp_weighted (the caller's weights, gi_graph_csr's edge order) == Dijkstra on the
    oracle's graph: random weights in [0, 1000] (zeros included), heavy-tailed weights, and
    graphgen's weights (which must also reproduce gi_sssp with that seed)."""
    import torch

    cfg = graphgen.CONFIGS[1]
    s1, d1 = cfg.edges()
    s3, d3 = graphgen.grid(64, 64, 0.2, 9)
    cases = [("config1", cfg.n, s1, d1, False, [0, 5]), ("config1-sym", cfg.n, s1, d1, True, [7]),
             ("grid64", 64 * 64, s3, d3, False, [0, 2000]),
             ("random", 3001, *graphgen.random_digraph(3001, 30000, 5), False, [0, 3000])]
    rng = np.random.default_rng(11)
    for name, n, s, d, sym, srcs in cases:
        flags = gi.GI_DEFAULT_FLAGS | (gi.GI_SYMMETRIZE if sym else 0)
        g = gi.Graph(ctx, n, s, d, flags)
        go = oracle.build_graph(n, s, d, symmetrize=sym)
        off, idx = g.csr()
        assert np.array_equal(off, go.csr_off) and np.array_equal(idx, go.csr_idx)  # the documented order
        for kind in ("uniform", "heavy", "graphgen"):
            if kind == "uniform":
                w = rng.integers(0, 1001, go.m).astype(np.int32)
            elif kind == "heavy":
                w = np.minimum(rng.pareto(1.2, go.m) * 50, 1e6).astype(np.int32)
            else:
                w = oracle.csr_weights(go, 5)
            for src in srcs:
                want = oracle.sssp(go, src, w)
                for where in ("host", "device"):
                    ww = w if where == "host" else torch.from_numpy(w).cuda()
                    got, _ = g.sssp_weighted(src, ww, policy=_pol(gi, policy))
                    assert (got.astype(np.int64) == want).all(), \
                        f"{name} {kind} src={src} {policy} {where}: {int((got != want).sum())} differ"
                if kind == "graphgen":
                    got2, _ = g.sssp(src, seed=5, policy=_pol(gi, policy))
                    assert (got2.astype(np.int64) == want).all()
        bad = np.zeros(go.m, np.int32)
        bad[go.m // 2] = -1
        with pytest.raises(gi.GiError):
            g.sssp_weighted(0, bad)
        with pytest.raises(ValueError):
            g.sssp_weighted(0, bad[:-1])
        g.close()


def test_sssp_device_output_and_errors(gi, ctx):
    import torch

    s, d = graphgen.rmat(12, 8, 0.57, 0.19, 0.19, 4)
    n = 1 << 12
    g = gi.Graph(ctx, n, s, d)
    go = oracle.build_graph(n, s, d)
    want = oracle.sssp(go, 0, oracle.csr_weights(go, 5))
    out = torch.full((n,), -9, dtype=torch.int32, device="cuda")
    got, st = g.sssp(0, seed=5, out=out, profile=True)
    assert (got.cpu().numpy().astype(np.int64) == want).all()
    assert st.total_ms > 0 and st.rounds >= 1
    with pytest.raises(gi.GiError) as e:
        g.sssp(n)
    assert e.value.status == gi.GI_ERR_VERTEX_OUT_OF_RANGE


def test_cc_pr_share_the_segmented_layout(gi, ctx):
    """CC's min passes and PageRank's sum passes run on the same segmented layout
    (whichever call builds it first) and on separate accumulators: interleaved
    calls on one graph keep both exact."""
    s, d = graphgen.rmat(17, 16, 0.57, 0.19, 0.19, 8)
    n = 1 << 17
    g = gi.Graph(ctx, n, s, d, gi.GI_DEFAULT_FLAGS | gi.GI_SYMMETRIZE)
    go = oracle.build_graph(n, s, d, symmetrize=True)
    want_cc = oracle.cc_labels(go)
    want_pr = oracle.pagerank(go, 20, 0.85)
    for step in range(2):
        lab, _ = g.cc()  # step 0: builds the layout
        assert (lab == want_cc).all(), step
        pr, _ = g.pagerank(20, 0.85)
        pr = np.asarray(pr, np.float64)
        assert np.abs(pr - want_pr).sum() <= 1e-5 and (np.abs(pr - want_pr) / want_pr).max() <= 1e-4, step
        par, _ = g.bfs_multi(graphgen.pick_sources(n, s, d, 8, step).tolist())  # AUTO: bit-parallel
        assert par.shape == (8, n)


def _pieces_model(n, s, d, Z):
    """The segmented layout's piece count from the edge list alone (test-side model, not the
    method): vertices relabelled by descending count of edge-list entries per source (ties by id,
    duplicates and self-loops counted), the cleaned edges' (source segment, destination) pairs."""
    s = np.asarray(s, np.int64)
    d = np.asarray(d, np.int64)
    cnt = np.bincount(s, minlength=n)
    order = np.lexsort((np.arange(n), -cnt))
    new = np.empty(n, np.int64)
    new[order] = np.arange(n)
    keep = s != d
    key = np.unique(new[d[keep]] * n + new[s[keep]])  # cleaned edges (destination, source)
    return int(np.unique((key % n) // Z * n + key // n).size)


def test_pr_segmented_reductions_per_iter(gi, ctx):
    """gi_pr_stats.reductions_per_iter (the bench's atomics bound) is exactly one RED per
    (source segment, destination row) pair with an edge, whatever the
    destination blocking; the record stream is whole records."""
    cfg = graphgen.CONFIGS[1]
    s, d = cfg.edges()
    g = gi.Graph(ctx, cfg.n, s, d)
    m = oracle.build_graph(cfg.n, s, d).m
    for Z, dblk in ((1000, 0), (1000, 4096), (4096, 0), (40000, 20000)):
        _, st = g.pagerank(2, 0.85, direction=gi.GI_PR_PULL_SEGMENTED, segment_size=Z, dst_block=dblk)
        assert st.kernel == gi.GI_PR_PULL_SEGMENTED
        assert st.reductions_per_iter == _pieces_model(cfg.n, s, d, Z), (Z, dblk)
        assert st.stream_bytes_per_iter > 0 and st.stream_bytes_per_iter % 1184 == 0
        assert st.stream_bytes_per_iter >= 2 * m  # 2-byte in-segment source indices at least
    _, st = g.pagerank(2, 0.85, direction=gi.GI_PR_PULL_DIRECT)
    assert st.reductions_per_iter == 0 and st.stream_bytes_per_iter == 0
    g.close()

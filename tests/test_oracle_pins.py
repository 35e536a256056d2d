"""Pins for the CPU oracle (`oracle/`): closed forms, invariants, brute force.

Each pin is independent of the oracle's own formulation (a different
formulation, a textbook routine on a special case, or a property), chosen so
that a dropped term, wrong sign/index or transposed operand fails one of them:

* PageRank
  - directed n-cycle and complete digraph K_n: r = 1/n (symmetry)
  - bidirectional star: exact closed form at k (tests/golden/pr_star_closed_form.json)
    -> pins the r[u]/outdeg(u) edge weight and where d multiplies
  - in-star (centre dangling): mass conservation (uniform rule) and the
    drop-rule mass recurrence -> pins the D_k term and its rule
  - exhaustive digraphs n <= 3 (20 iters) / n = 4 (4 iters) with exact
    rationals in the affine MATRIX form r' = M r + (1-d)/n (not the oracle's
    per-row loop)
  - random digraphs 5 <= n <= 8: matrix power in fp64
  - stationary limit = principal eigenvector of the Google matrix (numpy.linalg.eig)
* BFS
  - path (golden S:509), star, K_n, undropped grid depth = r + c, reverse-only
    edge, disconnected, Floyd-Warshall brute force on n <= 8
  - validator vs. exhaustive enumeration of parent vectors with a walk-based
    definition of a shortest-path tree
  - level-synchronous depths (OpenMP, billion-edge configs) = the FIFO depths
  - TEPS count (R16) = sum of raw out-degrees over the Floyd-Warshall reachable set
* Build: edge set = numpy.unique of the cleaned pairs; CSC = transpose of CSR.
"""
from __future__ import annotations

import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import graphgen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _digraph_from_mask(n, mask):
    pairs = [(u, v) for u in range(n) for v in range(n) if u != v]
    src = [u for i, (u, v) in enumerate(pairs) if mask >> i & 1]
    dst = [v for i, (u, v) in enumerate(pairs) if mask >> i & 1]
    return np.array(src, np.int32), np.array(dst, np.int32)


def _affine_pr_exact(n, src, dst, iters, d: Fraction, uniform=True):
    """r_{k+1} = M r_k + (1-d)/n * 1 with M[v][u] = d*A[u][v]/outdeg(u)
    (+ d/n for dangling u under the uniform rule) — exact rationals."""
    A = [[0] * n for _ in range(n)]
    for u, v in zip(src.tolist(), dst.tolist()):
        A[u][v] = 1
    outdeg = [sum(A[u]) for u in range(n)]
    M = [[Fraction(0)] * n for _ in range(n)]
    for u in range(n):
        for v in range(n):
            if outdeg[u]:
                M[v][u] = d * Fraction(A[u][v], outdeg[u])
            elif uniform:
                M[v][u] = d / n
    r = [Fraction(1, n)] * n
    c = (1 - d) / n
    for _ in range(iters):
        r = [sum((M[v][u] * r[u] for u in range(n)), Fraction(0)) + c for v in range(n)]
    return r


# ---------------------------------------------------------------- PageRank pins
@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 1000])
def test_pr_cycle_uniform(n):
    s, d = graphgen.cycle(n)
    g = oracle.build_graph(n, s, d)
    for iters in (0, 1, 20):
        r = oracle.pagerank(g, iters, 0.85)
        np.testing.assert_allclose(r, 1.0 / n, rtol=1e-15, atol=0)


@pytest.mark.parametrize("n", [2, 5, 9])
def test_pr_complete_uniform(n):
    s, d = graphgen.complete(n)
    g = oracle.build_graph(n, s, d)
    np.testing.assert_allclose(oracle.pagerank(g, 20, 0.85), 1.0 / n, rtol=1e-14)


def _star_closed_form(L, d, k):
    n = L + 1
    d = Fraction(d)
    rc_star = (1 + d * L) / (n * (1 + d))
    rl_star = (1 - d) / n + d * rc_star / L
    ec0 = Fraction(1, n) - rc_star
    el0 = Fraction(1, n) - rl_star
    if k % 2 == 0:
        ec, el = d**k * ec0, d**k * el0
    else:
        ec, el = d**k * L * el0, d**k * ec0 / L
    return rc_star + ec, rl_star + el


def test_pr_star_closed_form():
    cases = json.load(open(os.path.join(GOLDEN, "pr_star_closed_form.json")))["cases"]
    for c in cases:
        L, dmp, k = c["leaves"], c["damping"], c["iters"]
        s, d = graphgen.star_bidirectional(L)
        g = oracle.build_graph(L + 1, s, d)
        r = oracle.pagerank(g, k, dmp)
        rc, rl = _star_closed_form(L, Fraction(dmp).limit_denominator(10**6), k)
        assert abs(r[0] - float(rc)) <= 1e-14 * float(rc), c
        np.testing.assert_allclose(r[1:], float(rl), rtol=1e-13)


def test_pr_star_closed_form_is_not_trivial():
    # the closed form must move away from 1/n, else the pin pins nothing
    rc, rl = _star_closed_form(10, Fraction(17, 20), 20)
    assert abs(float(rc) - 1 / 11) > 0.1


@pytest.mark.parametrize("L", [1, 4, 50])
def test_pr_in_star_mass(L):
    s, d = graphgen.in_star(L)
    n = L + 1
    g = oracle.build_graph(n, s, d)
    for k in range(0, 25):
        r = oracle.pagerank(g, k, 0.85, oracle.UNIFORM)
        assert abs(r.sum() - 1.0) < 1e-13
        assert r.min() >= 0.15 / n * (1 - 1e-12)
    # drop rule: sum r_{k+1} = (1-d) + d (sum r_k - D_k), D_k = r_k[centre]
    dmp = 0.85
    prev = oracle.pagerank(g, 0, dmp, oracle.DROP)
    for k in range(1, 12):
        cur = oracle.pagerank(g, k, dmp, oracle.DROP)
        expect = (1 - dmp) + dmp * (prev.sum() - prev[0])
        assert abs(cur.sum() - expect) < 1e-13
        prev = cur
    # and the two rules differ materially on a dangling-heavy graph
    assert abs(oracle.pagerank(g, 5, dmp).sum() - oracle.pagerank(g, 5, dmp, oracle.DROP).sum()) > 0.1


@pytest.mark.parametrize("n", [1, 2, 3])
def test_pr_exhaustive_small_exact_20(n):
    npairs = n * (n - 1)
    d = Fraction(17, 20)
    for mask in range(1 << npairs):
        s, t = _digraph_from_mask(n, mask)
        g = oracle.build_graph(n, s, t)
        for uniform in (True, False):
            exact = _affine_pr_exact(n, s, t, 20, d, uniform)
            r = oracle.pagerank(g, 20, 0.85, oracle.UNIFORM if uniform else oracle.DROP)
            np.testing.assert_allclose(r, [float(x) for x in exact], rtol=1e-14, atol=0)


def test_pr_exhaustive_n4_exact():
    n, d = 4, Fraction(17, 20)
    for mask in range(1 << 12):
        s, t = _digraph_from_mask(n, mask)
        g = oracle.build_graph(n, s, t)
        exact = _affine_pr_exact(n, s, t, 4, d, True)
        r = oracle.pagerank(g, 4, 0.85)
        np.testing.assert_allclose(r, [float(x) for x in exact], rtol=1e-14, atol=0)


def _affine_float(n, src, dst, d, uniform):
    A = np.zeros((n, n))
    A[src, dst] = 1.0
    outdeg = A.sum(1)
    M = np.zeros((n, n))
    for u in range(n):
        if outdeg[u] > 0:
            M[:, u] = d * A[u] / outdeg[u]
        elif uniform:
            M[:, u] = d / n
    return M


def test_pr_random_small_matrix_power():
    rng = np.random.default_rng(7)
    for trial in range(400):
        n = int(rng.integers(5, 9))
        m0 = int(rng.integers(0, n * n))
        s, t = graphgen.random_digraph(n, m0, 1000 + trial)
        g = oracle.build_graph(n, s, t)
        keep = s != t
        e = np.unique(np.stack([s[keep], t[keep]], 1), axis=0) if keep.any() else np.zeros((0, 2), int)
        for uniform in (True, False):
            M = _affine_float(n, e[:, 0], e[:, 1], 0.85, uniform)
            r = np.full(n, 1.0 / n)
            for _ in range(20):
                r = M @ r + 0.15 / n
            got = oracle.pagerank(g, 20, 0.85, oracle.UNIFORM if uniform else oracle.DROP)
            np.testing.assert_allclose(got, r, rtol=1e-12, atol=0)


def test_pr_stationary_is_principal_eigenvector():
    for trial in range(20):
        n = 8
        s, t = graphgen.random_digraph(n, 20, 50 + trial)
        g = oracle.build_graph(n, s, t)
        keep = s != t
        e = np.unique(np.stack([s[keep], t[keep]], 1), axis=0)
        G = _affine_float(n, e[:, 0], e[:, 1], 0.85, True) + 0.15 / n
        w, V = np.linalg.eig(G)
        x = np.real(V[:, np.argmax(np.real(w))])
        x = x / x.sum()
        np.testing.assert_allclose(oracle.pagerank(g, 300, 0.85), x, rtol=1e-10)


def test_pr_edge_cases():
    g = oracle.build_graph(5, np.zeros(0, np.int32), np.zeros(0, np.int32))
    np.testing.assert_allclose(oracle.pagerank(g, 20, 0.85), 0.2, rtol=1e-15)  # all dangling
    g0 = oracle.build_graph(0, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert oracle.pagerank(g0, 20, 0.85).shape == (0,)
    with pytest.raises(oracle.OracleError):
        oracle.pagerank(g, 20, 1.5)


# ---------------------------------------------------------------- BFS pins
def test_bfs_path_golden():
    gd = json.load(open(os.path.join(GOLDEN, "bfs_path4.json")))
    g = oracle.build_graph(gd["n"], np.array(gd["src"], np.int32), np.array(gd["dst"], np.int32))
    depth = oracle.bfs_depth(g, gd["source"])
    assert depth.tolist() == gd["depth"]
    ok, msg = oracle.validate_bfs(g, gd["source"], np.array(gd["parent"], np.int32), depth)
    assert ok, msg


def test_bfs_star_complete_reverse_disconnected():
    s, d = graphgen.star_bidirectional(6)
    g = oracle.build_graph(7, s, d)
    assert oracle.bfs_depth(g, 0).tolist() == [0] + [1] * 6
    assert oracle.bfs_depth(g, 3).tolist() == [1, 2, 2, 0, 2, 2, 2]
    s, d = graphgen.complete(6)
    g = oracle.build_graph(6, s, d)
    assert oracle.bfs_depth(g, 2).tolist() == [1, 1, 0, 1, 1, 1]
    g = oracle.build_graph(2, np.array([1], np.int32), np.array([0], np.int32))
    assert oracle.bfs_depth(g, 0).tolist() == [0, -1]
    g = oracle.build_graph(5, np.array([0, 1, 3], np.int32), np.array([1, 0, 4], np.int32))
    assert oracle.bfs_depth(g, 0).tolist() == [0, 1, -1, -1, -1]


def test_bfs_undropped_grid_depth_is_manhattan():
    R, C = 37, 23
    s, d = graphgen.grid(R, C, 0.0, 3)
    g = oracle.build_graph(R * C, s, d)
    depth = oracle.bfs_depth(g, 0)
    rr, cc = np.divmod(np.arange(R * C), C)
    assert np.array_equal(depth, rr + cc)


def _floyd_warshall(n, src, dst):
    INF = 10**9
    D = np.full((n, n), INF, np.int64)
    np.fill_diagonal(D, 0)
    for u, v in zip(src.tolist(), dst.tolist()):
        if u != v:
            D[u, v] = 1
    for k in range(n):
        D = np.minimum(D, D[:, [k]] + D[[k], :])
    D[D >= INF] = -1
    return D


def test_bfs_brute_force_small():
    for trial in range(300):
        n = 1 + trial % 8
        s, t = graphgen.random_digraph(n, (trial * 7) % (3 * n + 1), 9000 + trial)
        g = oracle.build_graph(n, s, t)
        D = _floyd_warshall(n, s, t)
        for src in range(n):
            assert oracle.bfs_depth(g, src).tolist() == D[src].tolist()
            assert oracle.bfs_depth_levels(g, src).tolist() == D[src].tolist()


def test_bfs_levels_equals_fifo_on_rmat():
    """or_bfs_depth_levels (OpenMP, level-synchronous) = the FIFO BFS on graphs with many levels
    and wide frontiers (RMAT, a ragged grid, a path)."""
    cases = [(1 << 12, *graphgen.rmat(12, 8, 0.57, 0.19, 0.19, 21)),
             (64 * 64, *graphgen.grid(64, 64, 0.3, 5)), (500, *graphgen.path(500))]
    for n, s, t in cases:
        g = oracle.build_graph(n, s, t)
        for src in [0, 1, n // 3, n - 1]:
            assert np.array_equal(oracle.bfs_depth_levels(g, src), oracle.bfs_depth(g, src)), (n, src)


def test_reached_out_edges_brute_force():
    """R16's TEPS count = sum of out-degrees (counted from the raw cleaned pairs) over the vertices
    Floyd-Warshall says are reachable."""
    for trial in range(200):
        n = 1 + trial % 8
        s, t = graphgen.random_digraph(n, (trial * 5) % (3 * n + 1), 7000 + trial)
        g = oracle.build_graph(n, s, t)
        D = _floyd_warshall(n, s, t)
        pairs = {(int(a), int(b)) for a, b in zip(s, t) if a != b}
        outdeg = [sum(1 for (a, _) in pairs if a == u) for u in range(n)]
        for src in range(n):
            want = sum(outdeg[v] for v in range(n) if D[src][v] >= 0)
            assert oracle.reached_out_edges(g, oracle.bfs_depth(g, src)) == want


def _walk_valid(n, edges, dist, s, parent):
    if parent[s] != s:
        return False
    for v in range(n):
        if v == s:
            continue
        if dist[v] < 0:
            if parent[v] != -1:
                return False
            continue
        x, steps = v, 0
        while x != s and steps <= n:
            p = parent[x]
            if p < 0 or (p, x) not in edges:
                return False
            x, steps = p, steps + 1
        if x != s or steps != dist[v]:
            return False
    return True


def test_validator_exhaustive_tiny():
    checked = 0
    for trial in range(12):
        n = 3 + trial % 2
        s, t = graphgen.random_digraph(n, 2 * n + trial % 3, 300 + trial)
        g = oracle.build_graph(n, s, t)
        edges = {(int(a), int(b)) for a, b in zip(s, t) if a != b}
        for src in range(n):
            dist = oracle.bfs_depth(g, src)
            for cand in itertools.product(range(-1, n), repeat=n):
                want = _walk_valid(n, edges, dist.tolist(), src, cand)
                got, _ = oracle.validate_bfs(g, src, np.array(cand, np.int32), dist)
                assert got == want, (n, src, cand)
                checked += want
    assert checked > 10  # some valid trees were actually exercised


def test_validator_rejects_corruptions():
    s, d = graphgen.rmat(10, 8, 0.57, 0.19, 0.19, 11)
    g = oracle.build_graph(1 << 10, s, d)
    depth = oracle.bfs_depth(g, 0)
    # construct one valid parent vector from the oracle graph (first in-neighbour one level up)
    parent = np.full(g.n, -1, np.int32)
    parent[0] = 0
    for v in range(g.n):
        if depth[v] > 0:
            for u in g.csc_idx[g.csc_off[v]:g.csc_off[v + 1]]:
                if depth[u] == depth[v] - 1:
                    parent[v] = u
                    break
    assert oracle.validate_bfs(g, 0, parent, depth)[0]
    reached = np.nonzero(depth > 1)[0]
    v = int(reached[0])
    bad = parent.copy(); bad[0] = -1
    assert not oracle.validate_bfs(g, 0, bad, depth)[0]
    bad = parent.copy(); bad[v] = v
    assert not oracle.validate_bfs(g, 0, bad, depth)[0]
    bad = parent.copy(); bad[v] = 0  # 0 is two levels up: not adjacent/not depth-1
    assert not oracle.validate_bfs(g, 0, bad, depth)[0]
    unreached = np.nonzero(depth < 0)[0]
    if len(unreached):
        bad = parent.copy(); bad[unreached[0]] = 0
        assert not oracle.validate_bfs(g, 0, bad, depth)[0]


# ---------------------------------------------------------------- build pins
def test_build_matches_numpy_unique():
    for seed, flags in [(1, (True, True, False)), (2, (True, True, True)), (3, (False, False, False)),
                        (4, (True, False, False))]:
        n = 300
        s, t = graphgen.random_digraph(n, 5000, seed)
        rm, dd, sym = flags
        g = oracle.build_graph(n, s, t, remove_self_loops=rm, dedup=dd, symmetrize=sym)
        a, b = s.astype(np.int64), t.astype(np.int64)
        if rm:
            k = a != b
            a, b = a[k], b[k]
        if sym:
            a, b = np.concatenate([a, b]), np.concatenate([b, a])
        pairs = np.stack([a, b], 1)
        pairs = np.unique(pairs, axis=0) if dd else pairs[np.lexsort((b, a))]
        assert g.m == len(pairs)
        got = np.stack([np.repeat(np.arange(n), np.diff(g.csr_off)), g.csr_idx], 1)
        assert np.array_equal(got, pairs)
        # CSC is the transpose of CSR
        gotc = np.stack([g.csc_idx, np.repeat(np.arange(n), np.diff(g.csc_off))], 1)
        assert np.array_equal(gotc[np.lexsort((gotc[:, 1], gotc[:, 0]))], pairs)
        assert g.outdeg.sum() == g.m and g.indeg.sum() == g.m
        if dd:
            for u in range(n):
                row = g.csr_idx[g.csr_off[u]:g.csr_off[u + 1]]
                assert np.all(np.diff(row) > 0)


def test_build_matches_numpy_unique_rmat():
    """The same pin on a skewed graph large enough for every thread to hold pairs of every key range."""
    n = 1 << 14
    s, t = graphgen.rmat(14, 16, 0.57, 0.19, 0.19, 31)
    for sym in (False, True):
        g = oracle.build_graph(n, s, t, symmetrize=sym)
        a, b = s.astype(np.int64), t.astype(np.int64)
        k = a != b
        a, b = a[k], b[k]
        if sym:
            a, b = np.concatenate([a, b]), np.concatenate([b, a])
        key = np.unique(a * n + b)
        assert g.m == len(key)
        assert np.array_equal(np.repeat(np.arange(n), np.diff(g.csr_off)) * n + g.csr_idx, key)
        keyt = np.sort(b * n + a)
        keyt = np.unique(keyt)
        assert np.array_equal(np.repeat(np.arange(n), np.diff(g.csc_off)) * n + g.csc_idx, keyt)


def test_build_out_of_range():
    with pytest.raises(oracle.OracleError):
        oracle.build_graph(3, np.array([0, 3], np.int32), np.array([1, 1], np.int32))
    with pytest.raises(oracle.OracleError):
        oracle.build_graph(3, np.array([0, -1], np.int32), np.array([1, 1], np.int32))


# ---------------------------------------------------------------- PageRankDelta pins
def test_prdelta_eps0_is_pagerank_drop_rule():
    """With eps = 0 every vertex with a nonzero delta propagates, and by linearity
    Rank_k = r_k of Jacobi PageRank under the drop rule (no dangling term):
    round 1 gives r_1 and Delta_1 = r_1 - r_0; round k adds d * P Delta_{k-1} = r_k - r_{k-1}."""
    for seed, (n, m0) in enumerate([(50, 300), (300, 900), (1000, 8000)]):
        s, d = graphgen.random_digraph(n, m0, 70 + seed)
        g = oracle.build_graph(n, s, d)
        for k in (1, 2, 7, 15):
            np.testing.assert_allclose(oracle.pagerank_delta(g, k, 0.85, 0.0),
                                       oracle.pagerank(g, k, 0.85, oracle.DROP), rtol=1e-11, atol=1e-15)


def test_prdelta_huge_eps_stops_after_round_one():
    s, d = graphgen.random_digraph(200, 1500, 4)
    g = oracle.build_graph(200, s, d)
    r1 = oracle.pagerank(g, 1, 0.85, oracle.DROP)
    rk, fs = oracle.pagerank_delta(g, 6, 0.85, 1e30, return_frontiers=True)
    np.testing.assert_allclose(rk, r1, rtol=1e-14)
    assert fs[0] == 200 and fs[1:].sum() == 0  # round 1 from all vertices, then nothing is active


def test_prdelta_cycle_symmetry_and_frontier_shrinks():
    s, d = graphgen.cycle(3)  # all ranks equal by symmetry
    g = oracle.build_graph(3, s, d)
    r = oracle.pagerank_delta(g, 10, 0.85, 0.1)
    assert np.ptp(r) == 0.0
    s, d = graphgen.rmat(12, 8, 0.57, 0.19, 0.19, 3)
    g = oracle.build_graph(1 << 12, s, d)
    r, fs = oracle.pagerank_delta(g, 12, 0.85, 0.1, return_frontiers=True)
    assert fs[0] == 1 << 12 and fs[-1] < fs[1]  # the active set shrinks as ranks converge
    rpr = oracle.pagerank(g, 12, 0.85, oracle.DROP)
    assert np.abs(r - rpr).sum() < 0.05 * rpr.sum()  # an approximation of PageRank


# ---------------------------------------------------------------- connected components (NEXT #4)
def _cc_paper_rounds(n, src, dst):
    """The paper's CC program literally (P:3440-3472 [punt]): IDs[v] = v, frontier =
    all vertices, then rounds of edges.from(frontier).apply(IDs[dst] min= IDs[src])
    .modified(IDs), synchronous (every edge reads the labels of the round's start),
    until the frontier is empty. Pure Python, small graphs only."""
    ids = list(range(n))
    frontier = set(range(n))
    edges = [(int(s), int(d)) for s, d in zip(src, dst)]
    rounds = 0
    while frontier:
        new = list(ids)
        for s, d in edges:
            if s in frontier and ids[s] < new[d]:
                new[d] = ids[s]
        frontier = {v for v in range(n) if new[v] != ids[v]}
        ids = new
        rounds += 1
    return np.array(ids, np.int32), rounds


def test_cc_closed_forms():
    n = 9
    path = (np.arange(n - 1, dtype=np.int32), np.arange(1, n, dtype=np.int32))
    g = oracle.build_graph(n, *path)
    assert (oracle.cc_labels(g) == 0).all()                     # 0 reaches everything
    g = oracle.build_graph(n, path[1], path[0])                   # reversed: nothing reaches v from below
    assert (oracle.cc_labels(g) == np.arange(n)).all()
    s, d = graphgen.cycle(n)
    assert (oracle.cc_labels(oracle.build_graph(n, s, d)) == 0).all()
    # two directed cycles {0..4}, {5..8} plus isolated 9, 10
    s = np.array([0, 1, 2, 3, 4, 5, 6, 7, 8], np.int32)
    d = np.array([1, 2, 3, 4, 0, 6, 7, 8, 5], np.int32)
    lab = oracle.cc_labels(oracle.build_graph(11, s, d))
    assert lab.tolist() == [0] * 5 + [5] * 4 + [9, 10]
    # m = 0: every vertex is its own label
    assert oracle.cc_labels(oracle.build_graph(5, np.zeros(0, np.int32), np.zeros(0, np.int32))).tolist() == [0, 1, 2, 3, 4]


def test_cc_symmetric_matches_components():
    """On symmetric graphs the fixed point is the smallest vertex of each connected
    component: checked against scipy's connected_components (a library routine)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(1, 300))
        m = int(rng.integers(0, 2 * n + 1))
        s = rng.integers(0, n, m).astype(np.int32)
        d = rng.integers(0, n, m).astype(np.int32)
        g = oracle.build_graph(n, s, d, symmetrize=True)
        lab = oracle.cc_labels(g)
        a = coo_matrix((np.ones(m), (s, d)), shape=(n, n))
        nc, comp = connected_components(a, directed=True, connection="weak")
        want = np.full(nc, n, np.int64)
        np.minimum.at(want, comp, np.arange(n))
        assert (lab == want[comp]).all(), trial


def test_cc_directed_brute_force_and_paper_rounds():
    """Directed graphs: label[v] = min{u : u = v or u ->* v} from a Floyd-Warshall
    style boolean closure, and the paper's synchronous rounds reach the same
    labels."""
    rng = np.random.default_rng(12)
    for trial in range(120):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(0, n * n + 1))
        s = rng.integers(0, n, m).astype(np.int32)
        d = rng.integers(0, n, m).astype(np.int32)
        g = oracle.build_graph(n, s, d)
        lab = oracle.cc_labels(g)
        reach = np.eye(n, dtype=bool)
        reach[s, d] = True
        for k in range(n):
            reach |= reach[:, [k]] & reach[[k], :]
        want = np.array([min(u for u in range(n) if reach[u, v]) for v in range(n)], np.int32)
        assert (lab == want).all(), trial
        keep = s != d
        paper, _ = _cc_paper_rounds(n, s[keep], d[keep])
        assert (paper == want).all(), trial


# ---------------------------------------------------------------- SSSP (NEXT #4)
def _mix64(z):
    M = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_edge_weight_generator():
    """graphgen's synthetic weights: 1 + mix64(mix64(seed) + (u << 32 | v)) % 255 (R24),
    deterministic, in [1, 255], seed-dependent, direction-dependent."""
    rng = np.random.default_rng(3)
    u = rng.integers(0, 1 << 31, 500).astype(np.int32)
    v = rng.integers(0, 1 << 31, 500).astype(np.int32)
    w = graphgen.edge_weights(9, u, v)
    want = [1 + (_mix64((_mix64(9) + ((int(a) << 32) | int(b))) & ((1 << 64) - 1)) % 255) for a, b in zip(u, v)]
    assert w.tolist() == want
    assert w.min() >= 1 and w.max() <= 255
    assert (graphgen.edge_weights(10, u, v) != w).mean() > 0.9
    assert (graphgen.edge_weights(9, v, u) != w).mean() > 0.9


def _bellman_ford_paper(n, src, dst, w, source):
    """The paper's SSSP literally: frontier-based Bellman-Ford, synchronous
    rounds of edges.from(frontier).apply(dist[dst] min= dist[src] + w).modified(dist)."""
    INF = float("inf")
    dist = [INF] * n
    dist[source] = 0
    frontier = {source}
    while frontier:
        new = list(dist)
        for s, d, ww in zip(src, dst, w):
            if s in frontier and dist[s] + ww < new[d]:
                new[d] = dist[s] + ww
        frontier = {v for v in range(n) if new[v] != dist[v]}
        dist = new
    return [(-1 if x == INF else int(x)) for x in dist]


def test_sssp_unit_weights_are_bfs_depths():
    for seed in range(6):
        s, d = graphgen.random_digraph(200, 700, seed)
        g = oracle.build_graph(200, s, d)
        for src in (0, 17, 199):
            dist = oracle.sssp(g, src, np.ones(g.m, np.int32))
            assert (dist == oracle.bfs_depth(g, src)).all()


def test_sssp_weighted_path_closed_form():
    n = 12
    s, d = graphgen.path(n)
    g = oracle.build_graph(n, s, d)
    w = np.arange(1, g.m + 1, dtype=np.int32)  # edge k -> k+1 weighs k+1
    dist = oracle.sssp(g, 0, w)
    assert dist.tolist() == [k * (k + 1) // 2 for k in range(n)]
    dist = oracle.sssp(g, 5, w)
    assert dist.tolist() == [-1] * 5 + [sum(range(6, 6 + j)) for j in range(n - 5)]


def test_sssp_brute_force_and_paper_rounds():
    """Tiny weighted digraphs: min-plus closure (Floyd-Warshall) and the paper's
    frontier Bellman-Ford give the oracle's distances."""
    rng = np.random.default_rng(13)
    for trial in range(100):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(0, n * n + 1))
        s = rng.integers(0, n, m).astype(np.int32)
        d = rng.integers(0, n, m).astype(np.int32)
        g = oracle.build_graph(n, s, d)
        w = oracle.csr_weights(g, trial)
        rows = np.repeat(np.arange(n), np.diff(g.csr_off))
        D = np.full((n, n), np.inf)
        np.fill_diagonal(D, 0)
        for a, b, ww in zip(rows, g.csr_idx, w):
            D[a, b] = min(D[a, b], ww)
        for k in range(n):
            D = np.minimum(D, D[:, [k]] + D[[k], :])
        for src in range(n):
            dist = oracle.sssp(g, src, w)
            want = np.where(np.isinf(D[src]), -1, D[src]).astype(np.int64)
            assert (dist == want).all(), trial
            assert dist.tolist() == _bellman_ford_paper(n, rows.tolist(), g.csr_idx.tolist(), w.tolist(), src)

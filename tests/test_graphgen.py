"""Input generator checks (graphgen is shared input infrastructure)."""
import numpy as np

import graphgen


def test_rmat_count_and_determinism():
    s, d = graphgen.rmat(12, 16, 0.57, 0.19, 0.19, 1)
    assert len(s) == 16 * 4096
    s2, d2 = graphgen.rmat(12, 16, 0.57, 0.19, 0.19, 1)
    assert np.array_equal(s, s2) and np.array_equal(d, d2)
    # counter-based: any window of the stream reproduces in isolation
    s3, d3 = graphgen.rmat(12, 16, 0.57, 0.19, 0.19, 1, first=1000, count=777)
    assert np.array_equal(s3, s[1000:1777]) and np.array_equal(d3, d[1000:1777])
    s4, _ = graphgen.rmat(12, 16, 0.57, 0.19, 0.19, 2)
    assert not np.array_equal(s, s4)
    assert s.min() >= 0 and s.max() < 4096 and d.min() >= 0 and d.max() < 4096


def test_rmat_quadrant_frequencies():
    scale, ef = 14, 16
    a, b, c = 0.57, 0.19, 0.19
    s, d = graphgen.rmat(scale, ef, a, b, c, 5)
    m = len(s)
    for bit in (scale - 1, 0, scale // 2):
        sb = (s >> bit) & 1
        db = (d >> bit) & 1
        for frac, p in [(sb.mean(), c + 0.05), (db.mean(), b + 0.05),
                        ((sb & db).mean(), 0.05), (((1 - sb) & (1 - db)).mean(), a)]:
            sigma = np.sqrt(p * (1 - p) / m)
            assert abs(frac - p) < 5 * sigma, (bit, frac, p)


def test_grid_structure():
    R, C = 64, 48
    s, d = graphgen.grid(R, C, 0.0, 1)
    assert len(s) == 2 * (R * (C - 1) + (R - 1) * C)
    diff = np.abs(s.astype(np.int64) - d)
    assert set(np.unique(diff).tolist()) == {1, C}
    s, d = graphgen.grid(R, C, 0.1, 3)
    und = R * (C - 1) + (R - 1) * C
    kept = len(s) // 2
    p = 0.9
    assert abs(kept - p * und) < 5 * np.sqrt(und * p * (1 - p))
    # both directions present for every kept edge
    fwd = set(zip(s.tolist(), d.tolist()))
    assert all((v, u) in fwd for u, v in fwd)


def test_config3_corner_not_isolated():
    cfg = graphgen.CONFIGS[3]
    # only the first row/column edges of the corner matter: edge k=0 (0->1) and vertical k=nh (0->C)
    nh = cfg.rows * (cfg.cols - 1)
    kept0 = graphgen.uniform(cfg.seed, 0) >= cfg.p_drop
    kept1 = graphgen.uniform(cfg.seed, nh) >= cfg.p_drop
    assert kept0 or kept1


def test_pick_sources():
    s, d = graphgen.rmat(10, 4, 0.57, 0.19, 0.19, 3)
    src = graphgen.pick_sources(1024, s, d, 16, 77)
    assert len(src) == 16 and len(set(src.tolist())) == 16
    has_out = set(s[s != d].tolist())
    assert all(int(v) in has_out for v in src)
    assert np.array_equal(src, graphgen.pick_sources(1024, s, d, 16, 77))


def test_checksum_order_independent():
    s, d = graphgen.rmat(10, 4, 0.57, 0.19, 0.19, 3)
    p = np.random.default_rng(0).permutation(len(s))
    assert graphgen.edge_checksum(s, d) == graphgen.edge_checksum(s[p], d[p])
    assert graphgen.edge_checksum(s, d) != graphgen.edge_checksum(d, s)

"""CPU oracle for the edgeset.apply hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package. The product path
(`paper_1805_00923_b200`) never imports it and shares no code with it.

All arithmetic lives in `gi_oracle.c` (plain C, fp64 PageRank and
PageRankDelta, FIFO BFS, Graph500-style validator); see its header for the PAPER.md passages each
function follows. This module only marshals numpy arrays.

Pins: tests/test_oracle_pins.py (closed forms, invariants, brute force).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gi_oracle.c")
_LIB = os.path.join(_HERE, "libgi_oracle.so")
_lock = threading.Lock()
_lib = None

UNIFORM, DROP = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle in-tree with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
            i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
            f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
            vp = ctypes.c_void_p
            lib.or_build.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
            lib.or_build.restype = ctypes.c_int64
            lib.or_graph_arrays.argtypes = [vp, i64p, i32p, i64p, i32p]
            lib.or_graph_arrays.restype = None
            lib.or_graph_free.argtypes = [vp]
            lib.or_graph_free.restype = None
            lib.or_pagerank.argtypes = [vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, f64p]
            lib.or_pagerank.restype = ctypes.c_int
            lib.or_bfs_depth.argtypes = [vp, ctypes.c_int32, i32p]
            lib.or_bfs_depth.restype = ctypes.c_int
            lib.or_bfs_depth_levels.argtypes = [vp, ctypes.c_int32, i32p]
            lib.or_bfs_depth_levels.restype = ctypes.c_int
            lib.or_validate_bfs.argtypes = [vp, ctypes.c_int32, i32p, i32p,
                                            ctypes.POINTER(ctypes.c_int64)]
            lib.or_validate_bfs.restype = ctypes.c_int
            lib.or_reached_out_edges.argtypes = [vp, i32p]
            lib.or_reached_out_edges.restype = ctypes.c_int64
            lib.or_pagerank_delta.argtypes = [vp, ctypes.c_int, ctypes.c_double, ctypes.c_double, f64p, vp]
            lib.or_pagerank_delta.restype = ctypes.c_int
            lib.or_cc_labels.argtypes = [vp, i32p]
            lib.or_cc_labels.restype = ctypes.c_int
            lib.or_sssp.argtypes = [vp, ctypes.c_int32, i32p, i64p]
            lib.or_sssp.restype = ctypes.c_int
            lib.or_set_threads.argtypes = [ctypes.c_int]
            lib.or_set_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def set_threads(t: int) -> int:
    """OpenMP threads of the oracle's loops (t <= 0: unchanged); returns the previous count."""
    return int(_get().or_set_threads(int(t)))


class OracleError(RuntimeError):
    pass


_VALIDATE_MSG = {
    1: "root is not its own parent",
    2: "reachability mismatch (parent -1 vs depth)",
    3: "parent out of range",
    4: "parent edge (parent[v], v) not in E",
    5: "depth(parent[v]) != depth(v) - 1",
}


@dataclass
class Graph:
    """Cleaned graph: V = {0..n-1}, CSR by source and CSC by destination."""

    n: int
    m: int
    csr_off: np.ndarray
    csr_idx: np.ndarray
    csc_off: np.ndarray
    csc_idx: np.ndarray
    _h: ctypes.c_void_p

    @property
    def outdeg(self) -> np.ndarray:
        return np.diff(self.csr_off).astype(np.int64)

    @property
    def indeg(self) -> np.ndarray:
        return np.diff(self.csc_off).astype(np.int64)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _get().or_graph_free(h)
            self._h = None


def build_graph(n: int, src, dst, remove_self_loops: bool = True, dedup: bool = True,
                symmetrize: bool = False) -> Graph:
    lib = _get()
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    if len(src) != len(dst):
        raise ValueError("src and dst lengths differ")
    h = ctypes.c_void_p()
    m = lib.or_build(n, len(src), src, dst, int(remove_self_loops), int(dedup), int(symmetrize),
                     ctypes.byref(h))
    if m == -2:
        raise OracleError("vertex out of range")
    if m < 0:
        raise OracleError(f"or_build failed ({m})")
    csr_off = np.empty(n + 1, np.int64)
    csc_off = np.empty(n + 1, np.int64)
    csr_idx = np.empty(m, np.int32)
    csc_idx = np.empty(m, np.int32)
    lib.or_graph_arrays(h, csr_off, csr_idx, csc_off, csc_idx)
    return Graph(n, int(m), csr_off, csr_idx, csc_off, csc_idx, h)


def pagerank(g: Graph, iters: int = 20, damping: float = 0.85, dangling: int = UNIFORM) -> np.ndarray:
    r = np.empty(max(g.n, 1), np.float64)
    rc = _get().or_pagerank(g._h, iters, damping, dangling, r)
    if rc != 0:
        raise OracleError(f"or_pagerank failed ({rc})")
    return r[: g.n]


def bfs_depth(g: Graph, source: int) -> np.ndarray:
    d = np.empty(max(g.n, 1), np.int32)
    rc = _get().or_bfs_depth(g._h, source, d)
    if rc != 0:
        raise OracleError(f"or_bfs_depth failed ({rc})")
    return d[: g.n]


def bfs_depth_levels(g: Graph, source: int) -> np.ndarray:
    """The same depths as bfs_depth, computed level by level with OpenMP (billion-edge configs)."""
    d = np.empty(max(g.n, 1), np.int32)
    rc = _get().or_bfs_depth_levels(g._h, source, d)
    if rc != 0:
        raise OracleError(f"or_bfs_depth_levels failed ({rc})")
    return d[: g.n]


def validate_bfs(g: Graph, source: int, parent, depth=None) -> tuple[bool, str]:
    """Graph500-style validation of a parent vector against oracle depths."""
    if depth is None:
        depth = bfs_depth(g, source)
    parent = np.ascontiguousarray(parent, np.int32)
    if parent.shape != (g.n,):
        return False, f"parent has shape {parent.shape}, expected ({g.n},)"
    bad = ctypes.c_int64(-1)
    rc = _get().or_validate_bfs(g._h, source, np.ascontiguousarray(depth, np.int32), parent,
                                ctypes.byref(bad))
    if rc == 0:
        return True, "ok"
    return False, f"{_VALIDATE_MSG.get(rc, rc)} at vertex {bad.value}"


def reached_out_edges(g: Graph, depth) -> int:
    return int(_get().or_reached_out_edges(g._h, np.ascontiguousarray(depth, np.int32)))


def pagerank_delta(g: Graph, iters: int = 10, damping: float = 0.85, epsilon: float = 0.1,
                   return_frontiers: bool = False):
    """PageRankDelta (readings R17, R18). Returns Rank (and the
    frontier size entering each round if return_frontiers)."""
    r = np.empty(max(g.n, 1), np.float64)
    fs = np.zeros(max(iters, 1), np.int64)
    rc = _get().or_pagerank_delta(g._h, iters, damping, epsilon, r, fs.ctypes.data)
    if rc != 0:
        raise OracleError(f"or_pagerank_delta failed ({rc})")
    return (r[: g.n], fs[:iters]) if return_frontiers else r[: g.n]


def cc_labels(g: Graph) -> np.ndarray:
    """Label propagation's fixed point (P:3440-3472 [punt]): label[v] = the
    smallest u with u = v or a directed path u ->* v (symmetric graph: the smallest
    vertex of v's component)."""
    out = np.empty(max(g.n, 1), np.int32)
    rc = _get().or_cc_labels(g._h, out)
    if rc != 0:
        raise OracleError(f"or_cc_labels failed ({rc})")
    return out[: g.n]


def sssp(g: Graph, source: int, w_csr) -> np.ndarray:
    """Shortest-path distances from source along out-edges, w_csr[j] = weight of CSR edge j
    (Dijkstra: the fixed point of the paper's frontier Bellman-Ford); -1 = unreachable."""
    w = np.ascontiguousarray(w_csr, np.int32)
    if w.shape != (g.m,):
        raise ValueError("one weight per CSR edge")
    dist = np.empty(max(g.n, 1), np.int64)
    rc = _get().or_sssp(g._h, source, w if g.m else np.zeros(1, np.int32), dist)
    if rc != 0:
        raise OracleError(f"or_sssp failed ({rc})")
    return dist[: g.n]


def csr_weights(g: Graph, seed: int) -> np.ndarray:
    """The synthetic weight (graphgen.edge_weights, input ids) of every CSR edge of g."""
    import graphgen

    rows = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(g.csr_off).astype(np.int64))
    return graphgen.edge_weights(seed, rows, g.csr_idx)

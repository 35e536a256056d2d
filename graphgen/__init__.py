"""Seeded synthetic inputs shared by the oracle tests, GPU parity tests and bench.

Input infrastructure only: this package emits edge lists and source lists and
holds none of the method's arithmetic (SURVEY §8(c) "Independence"). The C
core (`graphgen.c`) is compiled with gcc on first use (or by
`__graft_entry__.build()`).

Workload recipes mirror BASELINE.json `configs`:

=====  =============================================================  ==================
cfg    graph                                                          stands in for
=====  =============================================================  ==================
1      RMAT s16 ef16 a=.57 b=c=.19 d=.05, seed 1                        (parity config)
2      RMAT s22 ef16 same a/b/c/d, seed 2                               LiveJournal
3      4096x4096 grid, 4-nbr, 10% undirected edges dropped, seed 3      USAroad
4      RMAT s25 ef48 a=.57, seed 4                                      Twitter
5      RMAT s26 ef28 a=.45 b=c=.22 d=.11, symmetrised, seed 5           Friendster
=====  =============================================================  ==================

The paper's datasets are not in this container; the
synthetic configs stand in for them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "graphgen.c")
_LIB = os.path.join(_HERE, "libgraphgen.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile libgraphgen.so in-tree (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
            u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
            lib.gg_rmat.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, i32p, i32p]
            lib.gg_rmat.restype = None
            lib.gg_grid.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_void_p]
            lib.gg_grid.restype = ctypes.c_int64
            lib.gg_has_out_edge.argtypes = [ctypes.c_int64, ctypes.c_int64, i32p, i32p, u8p]
            lib.gg_has_out_edge.restype = None
            lib.gg_pick_sources.argtypes = [ctypes.c_int64, u8p, ctypes.c_int64, ctypes.c_uint64,
                                            ctypes.c_int64, i32p]
            lib.gg_pick_sources.restype = ctypes.c_int64
            lib.gg_edge_checksum.argtypes = [ctypes.c_int64, i32p, i32p]
            lib.gg_edge_checksum.restype = ctypes.c_uint64
            lib.gg_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
            lib.gg_uniform.restype = ctypes.c_double
            lib.gg_edge_weights.argtypes = [ctypes.c_uint64, ctypes.c_int64, i32p, i32p, i32p]
            lib.gg_edge_weights.restype = None
            _lib = lib
    return _lib


def uniform(seed: int, ctr: int) -> float:
    return _get().gg_uniform(seed, ctr)


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int,
         first: int = 0, count: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """RMAT edge stream [first, first+count) of ef * 2^scale edges (int32 src, dst)."""
    total = edge_factor * (1 << scale)
    if count is None:
        count = total - first
    src = np.empty(count, np.int32)
    dst = np.empty(count, np.int32)
    _get().gg_rmat(scale, a, b, c, seed, first, count, src, dst)
    return src, dst


def grid(rows: int, cols: int, p_drop: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """4-neighbour lattice with each undirected edge dropped with prob p_drop."""
    lib = _get()
    w = lib.gg_grid(rows, cols, p_drop, seed, None, None)
    src = np.empty(2 * w, np.int32)
    dst = np.empty(2 * w, np.int32)
    lib.gg_grid(rows, cols, p_drop, seed, src.ctypes.data, dst.ctypes.data)
    return src, dst


def pick_sources(n: int, src: np.ndarray, dst: np.ndarray, k: int, seed: int) -> np.ndarray:
    """k distinct vertices drawn uniformly from those with a non-self-loop out-edge."""
    lib = _get()
    elig = np.empty(max(n, 1), np.uint8)
    lib.gg_has_out_edge(n, len(src), np.ascontiguousarray(src, np.int32),
                        np.ascontiguousarray(dst, np.int32), elig)
    out = np.empty(max(k, 1), np.int32)
    got = lib.gg_pick_sources(n, elig, k, seed, max(64 * k, 1 << 20), out)
    return out[:got].copy()


def has_out_edge(n: int, src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """uint8[n]: 1 where v is the source of a non-self-loop pair of this edge list (or share of it)."""
    elig = np.empty(max(n, 1), np.uint8)
    _get().gg_has_out_edge(n, len(src), np.ascontiguousarray(src, np.int32), np.ascontiguousarray(dst, np.int32),
                           elig)
    return elig[:n]


def pick_sources_from_mask(n: int, eligible: np.ndarray, k: int, seed: int) -> np.ndarray:
    """pick_sources given the eligibility mask (e.g. OR-reduced over ranks holding shares of the edges)."""
    elig = np.ascontiguousarray(np.asarray(eligible) != 0, np.uint8)
    if len(elig) == 0:
        elig = np.zeros(1, np.uint8)
    out = np.empty(max(k, 1), np.int32)
    got = _get().gg_pick_sources(n, elig, k, seed, max(64 * k, 1 << 20), out)
    return out[:got].copy()


def edge_checksum(src: np.ndarray, dst: np.ndarray) -> int:
    return int(_get().gg_edge_checksum(len(src), np.ascontiguousarray(src, np.int32),
                                       np.ascontiguousarray(dst, np.int32)))


def edge_weights(seed: int, u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Synthetic integer weights in [1, 255] of the directed edges (u[i], v[i]) (input ids):
    1 + mix64(mix64(seed) + (u << 32 | v)) % 255 (SSSP inputs, reading R24)."""
    u = np.ascontiguousarray(u, np.int32)
    v = np.ascontiguousarray(v, np.int32)
    w = np.empty(len(u), np.int32)
    _get().gg_edge_weights(seed, len(u), u, v, w)
    return w


# ---------------------------------------------------------------- small families
def path(n: int) -> tuple[np.ndarray, np.ndarray]:
    s = np.arange(max(n - 1, 0), dtype=np.int32)
    return s, s + 1


def cycle(n: int) -> tuple[np.ndarray, np.ndarray]:
    s = np.arange(n, dtype=np.int32)
    return s, ((s + 1) % n).astype(np.int32)


def star_bidirectional(leaves: int) -> tuple[np.ndarray, np.ndarray]:
    """Centre 0, leaves 1..L, edges both ways."""
    lv = np.arange(1, leaves + 1, dtype=np.int32)
    z = np.zeros(leaves, np.int32)
    return np.concatenate([z, lv]), np.concatenate([lv, z])


def in_star(leaves: int) -> tuple[np.ndarray, np.ndarray]:
    """Leaves 1..L point at centre 0 (the only dangling vertex)."""
    lv = np.arange(1, leaves + 1, dtype=np.int32)
    return lv, np.zeros(leaves, np.int32)


def complete(n: int) -> tuple[np.ndarray, np.ndarray]:
    s, d = np.meshgrid(np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32), indexing="ij")
    keep = s != d
    return s[keep].ravel().astype(np.int32), d[keep].ravel().astype(np.int32)


def random_digraph(n: int, m: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """m pairs drawn uniformly (self-loops and duplicates included)."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, max(n, 1), m, dtype=np.int64).astype(np.int32),
            rng.integers(0, max(n, 1), m, dtype=np.int64).astype(np.int32))


# ---------------------------------------------------------------- BASELINE configs
@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    kind: str            # "rmat" | "grid"
    n: int
    scale: int = 0
    edge_factor: int = 0
    abcd: tuple = (0.57, 0.19, 0.19, 0.05)
    rows: int = 0
    cols: int = 0
    p_drop: float = 0.0
    seed: int = 0
    symmetrize: bool = False
    pr_iters: int = 20
    damping: float = 0.85
    bfs_sources: int = 1       # 0 -> vertex 0 / corner
    source_seed: int = 0

    def edges(self) -> tuple[np.ndarray, np.ndarray]:
        if self.kind == "rmat":
            a, b, c, _ = self.abcd
            return rmat(self.scale, self.edge_factor, a, b, c, self.seed)
        return grid(self.rows, self.cols, self.p_drop, self.seed)

    def sources(self, src: np.ndarray, dst: np.ndarray) -> np.ndarray:
        if self.source_seed == 0:
            return np.zeros(1, np.int32)
        return pick_sources(self.n, src, dst, self.bfs_sources, self.source_seed)


CONFIGS = {
    1: Config(1, "rmat-s16-ef16", "rmat", 1 << 16, scale=16, edge_factor=16, seed=1),
    2: Config(2, "rmat-s22-ef16", "rmat", 1 << 22, scale=22, edge_factor=16, seed=2,
              bfs_sources=64, source_seed=1002),
    3: Config(3, "grid-4096x4096-p0.1", "grid", 4096 * 4096, rows=4096, cols=4096, p_drop=0.1,
              seed=3),
    4: Config(4, "rmat-s25-ef48", "rmat", 1 << 25, scale=25, edge_factor=48, seed=4,
              bfs_sources=16, source_seed=1004),
    5: Config(5, "rmat-s26-ef28-sym", "rmat", 1 << 26, scale=26, edge_factor=28,
              abcd=(0.45, 0.22, 0.22, 0.11), seed=5, symmetrize=True, bfs_sources=16,
              source_seed=1005),
}


# ---------------------------------------------------------------- device generator (billion-edge configs)
_CU_SRC = os.path.join(_HERE, "graphgen_cuda.cu")
_CU_LIB = os.path.join(_HERE, "libgraphgen_cuda.so")
_cu = None


def build_cuda(force: bool = False) -> str:
    """Compile the CUDA twin of the RMAT generator (same counter-based stream)."""
    if force or not os.path.exists(_CU_LIB) or os.path.getmtime(_CU_LIB) < os.path.getmtime(_CU_SRC):
        tmp = _CU_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _CU_SRC])
        os.replace(tmp, _CU_LIB)
    return _CU_LIB


def rmat_device(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int, device: int = 0,
                first: int = 0, count: int | None = None):
    """RMAT edge stream [first, first+count) generated on the GPU into int32 torch tensors."""
    global _cu
    import torch

    with _lock:
        if _cu is None:
            lib = ctypes.CDLL(build_cuda())
            lib.gg_rmat_device.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]
            lib.gg_rmat_device.restype = ctypes.c_int
            _cu = lib
    total = edge_factor * (1 << scale)
    if count is None:
        count = total - first
    src = torch.empty(count, dtype=torch.int32, device=device)
    dst = torch.empty(count, dtype=torch.int32, device=device)
    rc = _cu.gg_rmat_device(scale, a, b, c, seed, first, count, src.data_ptr(), dst.data_ptr(),
                            torch.cuda.current_stream(device).cuda_stream)
    if rc != 0:
        raise RuntimeError(f"gg_rmat_device failed with CUDA error {rc}")
    return src, dst

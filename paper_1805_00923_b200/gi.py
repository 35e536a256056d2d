"""Thin ctypes binding of libgi.so — the C ABI in include/gi.h, same names.

Argument marshalling only: every step of the path runs in the CUDA library.
Arrays may be numpy arrays (host) or torch tensors (host or CUDA); the library
detects host vs device pointers itself. If libgi.so is missing this module
raises ImportError — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GI_LIBGI") or os.path.join(_PKG, "libgi.so")  # override: A/B experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1805_00923_b200.build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ constants (gi.h)
GI_OK = 0
GI_ERR_INVALID_ARGUMENT = 1
GI_ERR_VERTEX_OUT_OF_RANGE = 2
GI_ERR_OUT_OF_MEMORY = 3
GI_ERR_CUDA = 4
GI_ERR_NCCL = 5
GI_ERR_UNSUPPORTED = 6
GI_ERR_INTERNAL = 7

GI_EDGES_ON_DEVICE = 1 << 0
GI_REMOVE_SELF_LOOPS = 1 << 1
GI_DEDUP = 1 << 2
GI_SYMMETRIZE = 1 << 3
GI_NO_RELABEL = 1 << 4
GI_OFFSETS64 = 1 << 5
GI_DEFAULT_FLAGS = GI_REMOVE_SELF_LOOPS | GI_DEDUP

GI_PR_PULL, GI_PR_PUSH, GI_PR_PULL_DIRECT, GI_PR_PULL_SEGMENTED, GI_PR_PULL_PARTITIONED, GI_PR_PULL_BLOCKED = 0, 1, 2, 3, 4, 5
GI_DANGLING_UNIFORM, GI_DANGLING_DROP = 0, 1
GI_BFS_AUTO, GI_BFS_PUSH_ONLY, GI_BFS_PULL_ONLY = 0, 1, 2
GI_PRD_AUTO, GI_PRD_PUSH_ONLY, GI_PRD_PULL_ONLY = 0, 1, 2
GI_BFS_BATCH_AUTO, GI_BFS_BATCH_PER_SOURCE, GI_BFS_BATCH_BITPARALLEL = 0, 1, 2
GI_MS_PULL_AUTO, GI_MS_PULL_ROWS, GI_MS_PULL_SEGMENTED = 0, 1, 2


class gi_pr_opts(ctypes.Structure):
    _fields_ = [("direction", ctypes.c_int32), ("dangling", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("segment_size", ctypes.c_int32), ("dst_block", ctypes.c_int32)]


class gi_pr_stats(ctypes.Structure):
    _fields_ = [("edge_launches", ctypes.c_int32), ("aux_launches", ctypes.c_int32), ("edge_ms", ctypes.c_float),
                ("total_ms", ctypes.c_float), ("kernel", ctypes.c_int32), ("vertex_ms", ctypes.c_float),
                ("bytes_alg_per_iter", ctypes.c_int64), ("exchange", ctypes.c_int32), ("exchange_ms", ctypes.c_float),
                ("reductions_per_iter", ctypes.c_int64), ("stream_bytes_per_iter", ctypes.c_int64)]


GI_DT_INT32, GI_DT_INT64, GI_DT_F64 = 0, 1, 2
_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32)
_ALLGATHERV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.c_int32)
_ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                 ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32)


class gi_host_comm(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("allreduce", _ALLREDUCE_FN), ("allgatherv", _ALLGATHERV_FN),
                ("alltoallv", _ALLTOALLV_FN)]


class gi_prdelta_opts(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("threshold_div", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class gi_prdelta_stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int32), ("pull_rounds", ctypes.c_int32), ("active_total", ctypes.c_int64),
                ("total_ms", ctypes.c_float), ("launches", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class gi_bfs_opts(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("threshold_div", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("pull_kernel", ctypes.c_int32)]


class gi_cc_opts(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("threshold_div", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class gi_cc_stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int32), ("pull_rounds", ctypes.c_int32), ("edges_examined", ctypes.c_int64),
                ("total_ms", ctypes.c_float), ("launches", ctypes.c_int32)]


class gi_bfs_stats(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("pull_levels", ctypes.c_int32), ("reached", ctypes.c_int64),
                ("edges_traversed", ctypes.c_int64), ("total_ms", ctypes.c_float), ("launches", ctypes.c_int32),
                ("pull_ms", ctypes.c_float), ("edges_examined", ctypes.c_int64), ("pull_vertices", ctypes.c_int64),
                ("pull_edges_examined", ctypes.c_int64), ("pull_or_levels", ctypes.c_int32),
                ("pull_sparse_levels", ctypes.c_int32)]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_st = ctypes.c_int

_SIGS = {
    "gi_context_create": ([ctypes.c_int, _vp, ctypes.POINTER(_vp)], _st),
    "gi_nccl_unique_id": ([ctypes.c_char_p], _st),
    "gi_context_create_dist": ([ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                ctypes.POINTER(_vp)], _st),
    "gi_context_destroy": ([_vp], _st),
    "gi_context_rank": ([_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], _st),
    "gi_local_group_create": ([ctypes.c_int, ctypes.POINTER(_vp)], _st),
    "gi_local_group_destroy": ([_vp], _st),
    "gi_context_create_local": ([ctypes.c_int, _vp, _vp, ctypes.c_int, ctypes.POINTER(_vp)], _st),
    "gi_context_create_hostcomm": ([ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(gi_host_comm),
                                    ctypes.POINTER(_vp)], _st),
    "gi_partition_ranges": ([_i64, ctypes.c_int, _vp, _vp], _st),
    "gi_graph_partition": ([_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _st),
    "gi_graph_create": ([_vp, _i64, _i64, _vp, _vp, ctypes.c_uint32, ctypes.POINTER(_vp)], _st),
    "gi_graph_destroy": ([_vp], _st),
    "gi_graph_num_vertices": ([_vp, ctypes.POINTER(_i64)], _st),
    "gi_graph_num_edges": ([_vp, ctypes.POINTER(_i64)], _st),
    "gi_graph_out_degrees": ([_vp, _vp], _st),
    "gi_graph_in_degrees": ([_vp, _vp], _st),
    "gi_graph_csr": ([_vp, _vp, _vp], _st),
    "gi_pagerank": ([_vp, _i32, ctypes.c_double, _vp], _st),
    "gi_pagerank_ex": ([_vp, _i32, ctypes.c_double, ctypes.POINTER(gi_pr_opts), _vp,
                        ctypes.POINTER(gi_pr_stats)], _st),
    "gi_pagerank_delta": ([_vp, _i32, ctypes.c_double, ctypes.c_double, ctypes.POINTER(gi_prdelta_opts), _vp,
                           ctypes.POINTER(gi_prdelta_stats)], _st),
    "gi_bfs": ([_vp, _i32, _vp], _st),
    "gi_bfs_ex": ([_vp, _i32, ctypes.POINTER(gi_bfs_opts), _vp, ctypes.POINTER(gi_bfs_stats)], _st),
    "gi_cc": ([_vp, _vp], _st),
    "gi_sssp": ([_vp, _i32, ctypes.c_uint64, _vp], _st),
    "gi_sssp_ex": ([_vp, _i32, ctypes.c_uint64, ctypes.POINTER(gi_cc_opts), _vp, ctypes.POINTER(gi_cc_stats)], _st),
    "gi_sssp_weighted": ([_vp, _i32, _vp, ctypes.POINTER(gi_cc_opts), _vp, ctypes.POINTER(gi_cc_stats)], _st),
    "gi_cc_ex": ([_vp, ctypes.POINTER(gi_cc_opts), _vp, ctypes.POINTER(gi_cc_stats)], _st),
    "gi_bfs_multi": ([_vp, _i32, _vp, ctypes.POINTER(gi_bfs_opts), _vp, ctypes.POINTER(gi_bfs_stats)], _st),
    "gi_status_string": ([_st], ctypes.c_char_p),
    "gi_last_error": ([], ctypes.c_char_p),
    "gi_abi_version": ([], ctypes.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
GI_ABI_VERSION = 3  # include/gi.h: the struct layouts above
if _lib.gi_abi_version() != GI_ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI version {_lib.gi_abi_version()}, the binding {GI_ABI_VERSION}: rebuild it")


class GiError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.gi_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_lib.gi_status_string(status).decode()}: {msg}")


def _check(status: int, where: str) -> None:
    if status != GI_OK:
        raise GiError(status, where)


def _ptr(a, dtype) -> tuple[int, object]:
    """(address, keep-alive) of a contiguous numpy array or torch tensor of `dtype`."""
    if a is None:
        return 0, None
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=dtype)
        return a.ctypes.data, a
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        tdt = {np.int32: torch.int32, np.float32: torch.float32, np.int64: torch.int64}[dtype]
        if a.dtype != tdt or not a.is_contiguous():
            raise TypeError(f"tensor must be contiguous {tdt}, got {a.dtype}")
        return a.data_ptr(), a
    a = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return a.ctypes.data, a


# ------------------------------------------------------------------ C names
def gi_abi_version() -> int:
    return _lib.gi_abi_version()


def gi_context_create(device: int = 0, stream: int | None = None) -> int:
    out = _vp()
    _check(_lib.gi_context_create(device, stream or None, ctypes.byref(out)), "gi_context_create")
    return out.value


def gi_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.gi_nccl_unique_id(buf), "gi_nccl_unique_id")
    return buf.raw


def gi_context_create_dist(device: int, stream: int | None, rank: int, nranks: int, uid: bytes) -> int:
    out = _vp()
    _check(_lib.gi_context_create_dist(device, stream or None, rank, nranks, uid, ctypes.byref(out)),
           "gi_context_create_dist")
    return out.value


def gi_local_group_create(nranks: int) -> int:
    out = _vp()
    _check(_lib.gi_local_group_create(nranks, ctypes.byref(out)), "gi_local_group_create")
    return out.value


def gi_local_group_destroy(grp: int) -> None:
    _check(_lib.gi_local_group_destroy(grp), "gi_local_group_destroy")


def gi_context_create_local(device: int, stream: int | None, grp: int, rank: int) -> int:
    out = _vp()
    _check(_lib.gi_context_create_local(device, stream or None, grp, rank, ctypes.byref(out)),
           "gi_context_create_local")
    return out.value


def gi_context_create_hostcomm(device: int, stream: int | None, rank: int, nranks: int, comm) -> tuple[int, object]:
    """comm: an object with allreduce(buf: np.ndarray) (in-place sum; int32 / int64 / float64 view),
    allgatherv(buf: np.ndarray[uint8], off: list[int]) and alltoallv(send, soff, recv, roff) (uint8 views).
    Returns (context handle, keep-alive of the callback trampolines)."""
    dts = {GI_DT_INT32: np.int32, GI_DT_INT64: np.int64, GI_DT_F64: np.float64}

    def _u8(ptr, nbytes):
        return np.ctypeslib.as_array((ctypes.c_uint8 * max(int(nbytes), 1)).from_address(ptr))[: int(nbytes)] \
            if nbytes else np.empty(0, np.uint8)

    def ar(_u, buf, count, dtype):
        try:
            dt = dts[dtype]
            comm.allreduce(_u8(buf, count * np.dtype(dt).itemsize).view(dt))
            return 0
        except Exception:  # pragma: no cover - reported as GI_ERR_NCCL by the library
            return 1

    def ag(_u, buf, off, p):
        try:
            offs = [off[i] for i in range(p + 1)]
            comm.allgatherv(_u8(buf, offs[-1]), offs)
            return 0
        except Exception:  # pragma: no cover
            return 1

    def a2a(_u, send, soff, recv, roff, p):
        try:
            so = [soff[i] for i in range(p + 1)]
            ro = [roff[i] for i in range(p + 1)]
            comm.alltoallv(_u8(send, so[-1]), so, _u8(recv, ro[-1]), ro)
            return 0
        except Exception:  # pragma: no cover
            return 1

    cb = gi_host_comm(None, _ALLREDUCE_FN(ar), _ALLGATHERV_FN(ag), _ALLTOALLV_FN(a2a))
    out = _vp()
    _check(_lib.gi_context_create_hostcomm(device, stream or None, rank, nranks, ctypes.byref(cb), ctypes.byref(out)),
           "gi_context_create_hostcomm")
    return out.value, (cb, ar, ag, a2a, comm)


def gi_partition_ranges(n: int, nranks: int, weight_prefix) -> np.ndarray:
    pre = np.ascontiguousarray(weight_prefix, np.int64)
    if pre.shape != (n + 1,):
        raise ValueError("weight_prefix must have n + 1 entries")
    out = np.empty(nranks + 1, np.int64)
    _check(_lib.gi_partition_ranges(n, nranks, pre.ctypes.data, out.ctypes.data), "gi_partition_ranges")
    return out


def gi_graph_partition(g: int) -> tuple[int, int, int]:
    lo, hi, ml = _i64(), _i64(), _i64()
    _check(_lib.gi_graph_partition(g, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(ml)), "gi_graph_partition")
    return lo.value, hi.value, ml.value


def gi_context_destroy(ctx: int) -> None:
    _check(_lib.gi_context_destroy(ctx), "gi_context_destroy")


def gi_graph_create(ctx: int, n: int, src, dst, flags: int = GI_DEFAULT_FLAGS) -> int:
    ps, ks = _ptr(src, np.int32)
    pd, kd = _ptr(dst, np.int32)
    m0 = len(ks) if ks is not None else 0
    if (len(kd) if kd is not None else 0) != m0:
        raise ValueError("src and dst lengths differ")
    out = _vp()
    _check(_lib.gi_graph_create(ctx, n, m0, ps or None, pd or None, flags, ctypes.byref(out)), "gi_graph_create")
    return out.value


def gi_graph_destroy(g: int) -> None:
    _check(_lib.gi_graph_destroy(g), "gi_graph_destroy")


def gi_graph_num_vertices(g: int) -> int:
    v = _i64()
    _check(_lib.gi_graph_num_vertices(g, ctypes.byref(v)), "gi_graph_num_vertices")
    return v.value


def gi_graph_num_edges(g: int) -> int:
    v = _i64()
    _check(_lib.gi_graph_num_edges(g, ctypes.byref(v)), "gi_graph_num_edges")
    return v.value


def gi_graph_out_degrees(g: int, out=None):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    _check(_lib.gi_graph_out_degrees(g, p or None), "gi_graph_out_degrees")
    return keep


def gi_graph_in_degrees(g: int, out=None):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    _check(_lib.gi_graph_in_degrees(g, p or None), "gi_graph_in_degrees")
    return keep


def gi_graph_csr(g: int):
    n, m = gi_graph_num_vertices(g), gi_graph_num_edges(g)
    off = np.empty(n + 1, np.int64)
    idx = np.empty(max(m, 1), np.int32)
    _check(_lib.gi_graph_csr(g, off.ctypes.data, idx.ctypes.data), "gi_graph_csr")
    return off, idx[:m]


def gi_pagerank(g: int, iters: int, damping: float, out=None):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.float32)
    p, keep = _ptr(out, np.float32)
    _check(_lib.gi_pagerank(g, iters, damping, p or None), "gi_pagerank")
    return keep


def gi_pagerank_ex(g: int, iters: int, damping: float, out=None, direction: int = GI_PR_PULL,
                   dangling: int = GI_DANGLING_UNIFORM, profile: bool = False, segment_size: int = 0,
                   dst_block: int = 0):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.float32)
    p, keep = _ptr(out, np.float32)
    o = gi_pr_opts(direction, dangling, int(profile), segment_size, dst_block)
    s = gi_pr_stats()
    _check(_lib.gi_pagerank_ex(g, iters, damping, ctypes.byref(o), p or None, ctypes.byref(s)), "gi_pagerank_ex")
    return keep, s


def gi_pagerank_delta(g: int, iters: int, damping: float, epsilon: float, out=None, policy: int = GI_PRD_AUTO,
                      threshold_div: int = 0, profile: bool = False):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.float32)
    p, keep = _ptr(out, np.float32)
    o = gi_prdelta_opts(policy, threshold_div, int(profile), 0)
    s = gi_prdelta_stats()
    _check(_lib.gi_pagerank_delta(g, iters, damping, epsilon, ctypes.byref(o), p or None, ctypes.byref(s)),
           "gi_pagerank_delta")
    return keep, s


def gi_bfs(g: int, source: int, out=None):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    _check(_lib.gi_bfs(g, source, p or None), "gi_bfs")
    return keep


def gi_bfs_ex(g: int, source: int, out=None, policy: int = GI_BFS_AUTO, threshold_div: int = 0,
              profile: bool = False):
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    o = gi_bfs_opts(policy, threshold_div, int(profile), 0)
    s = gi_bfs_stats()
    _check(_lib.gi_bfs_ex(g, source, ctypes.byref(o), p or None, ctypes.byref(s)), "gi_bfs_ex")
    return keep, s


def gi_cc_ex(g: int, out=None, policy: int = GI_BFS_AUTO, threshold_div: int = 0, profile: bool = False):
    """Label-propagation components: out[v] = min input id u with u = v or u ->* v."""
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    o = gi_cc_opts(policy, threshold_div, int(profile), 0)
    s = gi_cc_stats()
    _check(_lib.gi_cc_ex(g, ctypes.byref(o), p or None, ctypes.byref(s)), "gi_cc_ex")
    return keep, s


def gi_sssp_ex(g: int, source: int, seed: int, out=None, policy: int = GI_BFS_AUTO, threshold_div: int = 0,
               profile: bool = False):
    """Shortest-path distances from source (frontier Bellman-Ford) with graphgen's synthetic weights
    of `seed`; -1 = unreachable."""
    n = gi_graph_num_vertices(g)
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    o = gi_cc_opts(policy, threshold_div, int(profile), 0)
    s = gi_cc_stats()
    _check(_lib.gi_sssp_ex(g, source, seed, ctypes.byref(o), p or None, ctypes.byref(s)), "gi_sssp_ex")
    return keep, s


def gi_sssp_weighted(g: int, source: int, weights, out=None, policy: int = GI_BFS_AUTO, threshold_div: int = 0,
                     profile: bool = False):
    """Shortest-path distances from source over caller weights: int32[m] in gi_graph_csr's edge order
    (input ids, rows and neighbours ascending), all >= 0; -1 = unreachable."""
    n, m = gi_graph_num_vertices(g), gi_graph_num_edges(g)
    pw, kw = _ptr(weights, np.int32)
    if (len(kw) if kw is not None else 0) != m:
        raise ValueError("one weight per edge of the cleaned graph")
    if out is None:
        out = np.empty(n, np.int32)
    p, keep = _ptr(out, np.int32)
    o = gi_cc_opts(policy, threshold_div, int(profile), 0)
    s = gi_cc_stats()
    _check(_lib.gi_sssp_weighted(g, source, pw or None, ctypes.byref(o), p or None, ctypes.byref(s)),
           "gi_sssp_weighted")
    return keep, s


def gi_bfs_multi(g: int, sources, out=None, policy: int = GI_BFS_AUTO, threshold_div: int = 0,
                 profile: bool = False, batch: int = GI_BFS_BATCH_AUTO, pull_kernel: int = GI_MS_PULL_AUTO):
    """k BFS runs back to back; out: int32[k, n] (host or device). Returns (out, [stats])."""
    n = gi_graph_num_vertices(g)
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).astype(np.int32))
    k = len(src)
    if out is None:
        out = np.empty((k, n), np.int32)
    p, keep = _ptr(out, np.int32)
    o = gi_bfs_opts(policy, threshold_div, int(profile), batch, pull_kernel)
    stats = (gi_bfs_stats * max(k, 1))()
    _check(_lib.gi_bfs_multi(g, k, src.ctypes.data if k else None, ctypes.byref(o), p or None, stats),
           "gi_bfs_multi")
    return keep, list(stats)[:k]


# ------------------------------------------------------------------ RAII conveniences
class Context:
    def __init__(self, device: int = 0, stream: int | None = None, *, local_group: int | None = None,
                 rank: int = 0, nccl: tuple | None = None, hostcomm: tuple | None = None):
        """local_group: simulated ranks in this process (tests); nccl: (rank, nranks, unique_id);
        hostcomm: (rank, nranks, comm) with comm as gi_context_create_hostcomm takes it."""
        import weakref

        self._keep = None
        if hostcomm is not None:
            self.handle, self._keep = gi_context_create_hostcomm(device, stream, hostcomm[0], hostcomm[1],
                                                                 hostcomm[2])
        elif local_group is not None:
            self.handle = gi_context_create_local(device, stream, local_group, rank)
        elif nccl is not None:
            self.handle = gi_context_create_dist(device, stream, nccl[0], nccl[1], nccl[2])
        else:
            self.handle = gi_context_create(device, stream)
        self._graphs = weakref.WeakSet()

    def close(self):
        """Destroys the context's live graphs first (the C ABI requires it)."""
        for g in list(getattr(self, "_graphs", ())):
            g.close()
        if self.handle:
            gi_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    def __init__(self, ctx: Context, n: int, src, dst, flags: int = GI_DEFAULT_FLAGS):
        self.ctx = ctx
        self.handle = None
        if not ctx.handle:
            raise GiError(GI_ERR_INVALID_ARGUMENT, "Graph: context is closed")
        self.handle = gi_graph_create(ctx.handle, n, src, dst, flags)
        ctx._graphs.add(self)
        self.n = gi_graph_num_vertices(self.handle)
        self.m = gi_graph_num_edges(self.handle)

    def close(self):
        if self.handle:
            gi_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def pagerank(self, iters=20, damping=0.85, out=None, **kw):
        return gi_pagerank_ex(self.handle, iters, damping, out, **kw)

    def pagerank_delta(self, iters=10, damping=0.85, epsilon=0.1, out=None, **kw):
        return gi_pagerank_delta(self.handle, iters, damping, epsilon, out, **kw)

    def bfs(self, source, out=None, **kw):
        return gi_bfs_ex(self.handle, source, out, **kw)

    def cc(self, out=None, **kw):
        return gi_cc_ex(self.handle, out, **kw)

    def sssp(self, source, seed=1, out=None, **kw):
        return gi_sssp_ex(self.handle, source, seed, out, **kw)

    def sssp_weighted(self, source, weights, out=None, **kw):
        return gi_sssp_weighted(self.handle, source, weights, out, **kw)

    def bfs_multi(self, sources, out=None, **kw):
        return gi_bfs_multi(self.handle, sources, out, **kw)

    def out_degrees(self, out=None):
        return gi_graph_out_degrees(self.handle, out)

    def in_degrees(self, out=None):
        return gi_graph_in_degrees(self.handle, out)

    def csr(self):
        return gi_graph_csr(self.handle)

    def partition(self):
        """(lo, hi, local_edges): owned destination range in internal ids."""
        return gi_graph_partition(self.handle)

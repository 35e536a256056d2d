"""Host-staged collectives for gi_context_create_hostcomm over torch.distributed.

Transport plumbing, not the hot path: the library stages each collective of
the multi-GPU path through host memory and calls these methods;
they run it on a torch.distributed process group with CPU tensors (gloo). Used
to run the destination-partitioned build / PageRank / BFS across processes
that share a GPU (tests) or where NCCL is not wanted.
"""
from __future__ import annotations

import numpy as np


class TorchDistComm:
    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce(self, buf: np.ndarray) -> None:
        import torch

        t = torch.from_numpy(buf.copy())
        self.dist.all_reduce(t, group=self.group)
        buf[:] = t.numpy()

    def _gather_bytes(self, mine: np.ndarray) -> list[np.ndarray]:
        """every rank's byte string (any lengths)."""
        import torch

        n = torch.tensor([len(mine)], dtype=torch.int64)
        lens = [torch.zeros(1, dtype=torch.int64) for _ in range(self.size)]
        self.dist.all_gather(lens, n, group=self.group)
        mx = max(1, max(int(x) for x in lens))
        pad = torch.zeros(mx, dtype=torch.uint8)
        pad[: len(mine)] = torch.from_numpy(mine.copy())
        outs = [torch.zeros(mx, dtype=torch.uint8) for _ in range(self.size)]
        self.dist.all_gather(outs, pad, group=self.group)
        return [o.numpy()[: int(k)] for o, k in zip(outs, lens)]

    def allgatherv(self, buf: np.ndarray, off: list[int]) -> None:
        parts = self._gather_bytes(buf[off[self.rank]: off[self.rank + 1]])
        for q, part in enumerate(parts):
            buf[off[q]: off[q + 1]] = part

    def alltoallv(self, send: np.ndarray, soff: list[int], recv: np.ndarray, roff: list[int]) -> None:
        sends = self._gather_bytes(send)
        soffs = self._gather_bytes(np.asarray(soff, np.int64).view(np.uint8))
        for q in range(self.size):
            so = soffs[q].view(np.int64)
            recv[roff[q]: roff[q + 1]] = sends[q][so[self.rank]: so[self.rank + 1]]

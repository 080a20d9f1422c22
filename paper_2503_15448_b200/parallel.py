"""Clients sharded across the GPUs of one node (one process per GPU).

The reference runs every client in one process (server.py:409-417 is the
only fan-out). Here each rank owns a fixed subset of clients, balanced by
longest-processing-time on their per-round SGD work, and trains only those.
A synchronous round then has exactly one exchange step:

    [ partial FedAvg sum (M, float64) | aligned counts (N) | accepted k | diverged (N) ]

packed into one float64 buffer and summed with a single NCCL all-reduce
(NVLink/NVSwitch on a B200 node). Every rank finishes the mean locally and
replays the same deterministic event loop from the reduced counts, so the
global model and the event log stay replicated without a broadcast.

Aggregation order: within a rank updates are summed in canonical byte
order; across ranks NCCL re-associates the sum, so G>1 results are
tolerance-matched to the single-GPU run (not bitwise). DESIGN.md §Multi-GPU.
"""

from __future__ import annotations

import heapq
import os

import numpy as np
import torch


def lpt_owner(work: np.ndarray, n_ranks: int) -> np.ndarray:
    """Rank owning each client: longest job first onto the least-loaded rank
    (ties by lower rank). Deterministic, identical on every rank."""
    work = np.asarray(work, dtype=np.float64)
    owner = np.zeros(len(work), dtype=np.int64)
    if n_ranks <= 1:
        return owner
    heap = [(0.0, r) for r in range(n_ranks)]
    for i in np.argsort(-work, kind="stable"):
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + float(work[i]), r))
    return owner


def client_work(world) -> np.ndarray:
    """Rows trained per round by each client: E * n_i (partial batches included)."""
    return np.array([world.epochs * wc.n for wc in world.clients], dtype=np.float64)


class RoundExchange:
    """Packs a rank's partial round results and all-reduces them in one call."""

    def __init__(self, M: int, N: int, device, group=None):
        self.M, self.N = M, N
        self.group = group
        self.buf = torch.zeros(M + 2 * N + 1, dtype=torch.float64, device=device)

    @property
    def partial_sum(self) -> torch.Tensor:
        """Slot the rank's partial FedAvg sum is written into (float64 [M])."""
        return self.buf[: self.M]

    def reduce(self, own_idx: np.ndarray, own_aligned: np.ndarray, own_diverged: np.ndarray, k_own: int):
        """All-reduce the packed buffer; returns (sum [M] view, aligned [N], k, diverged [N])."""
        import torch.distributed as dist

        M, N = self.M, self.N
        tail = np.zeros(2 * N + 1, dtype=np.float64)
        tail[np.asarray(own_idx, dtype=np.int64)] = np.asarray(own_aligned, dtype=np.float64)
        tail[N] = float(k_own)
        tail[N + 1 + np.asarray(own_idx, dtype=np.int64)] = np.asarray(own_diverged, dtype=np.float64)
        self.buf[M:].copy_(torch.from_numpy(tail), non_blocking=False)
        dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
        out = self.buf[M:].cpu().numpy()
        return self.buf[:M], out[:N].astype(np.int64), int(out[N]), out[N + 1:] != 0


class ShardComm:
    """Process-group plumbing for client sharding (torch.distributed)."""

    def __init__(self, rank: int, size: int, group=None):
        self.rank, self.size, self.group = rank, size, group

    @classmethod
    def from_env(cls) -> "ShardComm | None":
        size = int(os.environ.get("WORLD_SIZE", "1"))
        if size <= 1:
            return None
        import torch.distributed as dist

        if not dist.is_initialized():
            # FS_DIST_BACKEND=gloo lets several ranks share one GPU (tests)
            backend = os.environ.get("FS_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
            dist.init_process_group(backend)
        return cls(dist.get_rank(), dist.get_world_size())

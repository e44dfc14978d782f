"""Multi-GPU sharded scan: one process per GPU, contiguous sequence shards.

The paper's input partition (ingest.py:78-94) lifted to GPUs.  Each rank owns
the contiguous shard ``[begin, end)`` of the global sequence (resident in its
own HBM) and:

1. computes its shard's boundary map ``q -> state after the shard``
   (``ks_segment_map``: a constant for definite automata, a monoid element's
   action for map-scan automata; |Q| int32 = a few KB);
2. all-gathers the maps (NCCL over NVLink; gloo in the CPU tests) and composes
   the maps of ranks < r from START -> its true entry state (the reference's
   left-to-right chain, engine.py:155-163, over ranks);
3. scans its shard from that state on its GPU;
4. all-reduces the int64 per-expression counts.

Match rows stay sharded: offsets are global, so concatenating the ranks'
rows in rank order is the globally sorted list.  The scanner is injected so
the exchange logic is testable on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol

import numpy as np

START = 0


def shard_bounds(n: int, world: int, align: int = 64) -> list[tuple[int, int]]:
    """Contiguous shards covering [0, n), boundaries on `align`-base multiples."""
    if world < 1:
        raise ValueError("world must be >= 1")
    blocks = (n + align - 1) // align
    per, extra = divmod(blocks, world)
    bounds, b = [], 0
    for r in range(world):
        nb = per + (1 if r < extra else 0)
        e = min(n, (b + nb) * align) if r < world - 1 else n
        bounds.append((min(b * align, n), e))
        b += nb
    return bounds


def compose_entry(maps: np.ndarray, rank: int, start: int = START) -> int:
    """Entry state of `rank`: START pushed through the maps of ranks < rank."""
    s = start
    for r in range(rank):
        s = int(maps[r][s])
    return s


class ShardScanner(Protocol):
    n_states: int
    n_expressions: int

    def segment_map(self, begin: int, end: int) -> np.ndarray: ...

    def scan(self, begin: int, end: int, entry: int, locate: bool): ...


@dataclass
class DeviceShardScanner:
    """Scanner over a device-resident shard (positions local to the shard;
    ``row_base`` globalises row offsets)."""

    ctx: object
    dfa: object
    seq: object
    row_base: int = 0

    @property
    def n_states(self) -> int:
        return self.dfa.n_states

    @property
    def n_expressions(self) -> int:
        return self.dfa.n_expressions

    def segment_map(self, begin: int, end: int) -> np.ndarray:
        return self.ctx.segment_map(self.dfa, self.seq, begin, end)

    def scan(self, begin: int, end: int, entry: int, locate: bool):
        counts, _, rows = self.ctx.scan_range(self.dfa, self.seq, begin, end, entry, self.row_base, locate)
        return counts, rows


def run_sharded(scanner: ShardScanner, begin: int, end: int, group=None, locate: bool = False,
                device=None):
    """Steps 1-4 above for this rank's shard [begin, end) (local coordinates
    of ``scanner``).  Returns (global counts int64[ne], local rows | None)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1:
        counts, rows = scanner.scan(begin, end, START, locate)
        return counts, rows
    local_map = scanner.segment_map(begin, end).astype(np.int64)
    t = torch.from_numpy(local_map)
    if device is not None:
        t = t.to(device)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t, group=group)
    maps = np.stack([g.cpu().numpy() for g in gathered])
    entry = compose_entry(maps, rank)
    counts, rows = scanner.scan(begin, end, entry, locate)
    c = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64))
    if device is not None:
        c = c.to(device)
    dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
    return c.cpu().numpy(), rows

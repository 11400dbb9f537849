"""Frame sharding across ranks.

Per-frame work is independent given the stream's envelope, so a stream
of frames is cut into batches and round r gives batch r*world + rank to each
rank (no data-path collective).  The per-frame records (128 bytes each) are
all-gathered once per round; concatenated in rank order they are in frame
order, so every rank can run the sequential Mouse fold (a8) over them.

Pure host logic with injected callables, shared by bench.py (NCCL, libfizi)
and tests/test_multirank.py (gloo, CPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Batch:
    index: int      # batch number in the stream
    k0: int         # first frame (inclusive)
    k1: int         # last frame (exclusive)

    @property
    def n(self) -> int:
        return self.k1 - self.k0


def n_batches(n_frames: int, batch: int) -> int:
    return math.ceil(n_frames / batch)


def n_rounds(n_frames: int, batch: int, world: int) -> int:
    return math.ceil(n_batches(n_frames, batch) / world)


def round_batch(n_frames: int, batch: int, world: int, rank: int, rnd: int) -> Batch | None:
    """Batch rank `rank` processes in round `rnd` (rounds wrap), or None."""
    rnd %= n_rounds(n_frames, batch, world)
    b = rnd * world + rank
    if b >= n_batches(n_frames, batch):
        return None
    k0 = b * batch
    return Batch(b, k0, min(n_frames, k0 + batch))


def round_sizes(n_frames: int, batch: int, world: int, rnd: int) -> list[int]:
    """Frames each rank contributes in round `rnd` (0 for an idle rank)."""
    out = []
    for r in range(world):
        b = round_batch(n_frames, batch, world, r, rnd)
        out.append(b.n if b else 0)
    return out


def gathered_slices(n_frames: int, batch: int, world: int, rnd: int):
    """(offset, n) of each rank's records inside the gathered buffer of
    world * batch records, in frame order."""
    return [(r * batch, n) for r, n in enumerate(round_sizes(n_frames, batch, world, rnd)) if n]


def window_slices(n_frames: int, batch: int, world: int, rounds, window: int):
    """(offset, n) of the records, in frame order, inside the buffer gathered
    from every rank's window of `window` steps x `batch` records (rank r's
    block at r * window * batch, step j of the window at + j * batch);
    `rounds` are the rounds of the window's steps, in order."""
    out = []
    for j, rnd in enumerate(rounds):
        for off, n in gathered_slices(n_frames, batch, world, rnd):
            r = off // batch
            out.append((r * window * batch + j * batch, n))
    return out


# ------------------------------------------------ camera-stream sharding (C5)
# Many independent camera streams (BASELINE.json configs[4]): stream s lives
# on rank s mod world with its own envelope and tracker state, so no exchange
# is needed for correctness; each step the ranks all-gather the step's
# records (one per stream) for a global view.

def stream_shard(n_streams: int, world: int, rank: int) -> list[int]:
    """Global ids of the streams rank `rank` owns (s mod world == rank), in order;
    a stream's local id on its rank is its index in this list."""
    return list(range(rank, n_streams, world))


def streams_per_rank(n_streams: int, world: int) -> int:
    """Records each rank contributes per step to the gather (the largest shard;
    smaller shards pad)."""
    return math.ceil(n_streams / world)


def gathered_stream_ids(n_streams: int, world: int) -> list[int]:
    """Global stream id of every row of a gathered step buffer (world blocks of
    streams_per_rank rows, rank r's block first), -1 for padding rows."""
    per = streams_per_rank(n_streams, world)
    out = []
    for r in range(world):
        mine = stream_shard(n_streams, world, r)
        out.extend(mine + [-1] * (per - len(mine)))
    return out


def stream_order(n_streams: int, world: int) -> list[int]:
    """Row of the gathered step buffer holding global stream s, for s = 0..n-1."""
    ids = gathered_stream_ids(n_streams, world)
    pos = {s: i for i, s in enumerate(ids) if s >= 0}
    return [pos[s] for s in range(n_streams)]

"""Multi-GPU plumbing for batch decoding: one process per GPU (torchrun), frames
sharded across ranks, no exchange inside or between iterations (frames are
independent decoding problems).  After the timed region the per-rank error
counters are summed and the elapsed time maxed over ranks with
torch.distributed (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple


def frame_shard(rank: int, world: int, frames_per_rank: int) -> Tuple[int, int]:
    """Global frame range [f0, f0 + n) decoded by `rank` (weak scaling: every rank
    decodes `frames_per_rank` frames; global frame ids make the inputs independent
    of the number of ranks)."""
    if not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError("bad shard request")
    return rank * frames_per_rank, frames_per_rank


def reduce_counters(counters, elapsed_ms, group=None):
    """All-reduce error counters (SUM) and elapsed time (MAX) over the ranks.
    `counters` is an int64 tensor [bit_err, frame_err, undetected, not_converged,
    sum_iterations]; `elapsed_ms` a float64 tensor of shape [1].  In place; returns both."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(elapsed_ms, op=dist.ReduceOp.MAX, group=group)
    return counters, elapsed_ms


def count_errors_host(hard_bits_u32, syndrome_ok, iterations):
    """Host reference of ldpc_count_errors (all-zero codeword, reading D14): numpy arrays in,
    [bit_err, frame_err, undetected, not_converged, sum_iters] out."""
    import numpy as np
    hb = np.ascontiguousarray(hard_bits_u32).view(np.uint8)
    nbits = np.unpackbits(hb, axis=1).sum(axis=1).astype(np.int64)
    ok = np.asarray(syndrome_ok).astype(bool)
    return [int(nbits.sum()), int((nbits > 0).sum()), int(((nbits > 0) & ok).sum()), int((~ok).sum()),
            int(np.asarray(iterations, dtype=np.int64).sum())]

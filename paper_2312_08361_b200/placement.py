"""Which GPU serves which blocks.

The reference assigns spans on the host (`stage_intervals`, SP/swarm.py:40-49;
the Eq. 1 placement `choose_start`, SP/balancer.py:39-67).  The bench and the
multi-GPU pipeline need only the even split: rank r of N serves the r-th of N
contiguous spans whose sizes differ by at most one block, the larger spans
first.  For the configs of BASELINE.json this equals the reference's greedy
placement too (70B at 1/2/4/8 GPUs), which
tests/golden/assignment.json pins from the reference itself.
"""

from __future__ import annotations


def stage_intervals(n_blocks: int, n_stages: int) -> list[tuple[int, int]]:
    """[(start, end)] of `n_stages` contiguous spans tiling [0, n_blocks)."""
    if n_stages < 1 or n_blocks < n_stages:
        raise ValueError("need 1 <= n_stages <= n_blocks")
    size, rem = divmod(n_blocks, n_stages)
    bounds = [0]
    for r in range(n_stages):
        bounds.append(bounds[-1] + size + (r < rem))
    return list(zip(bounds[:-1], bounds[1:]))


def span_of_rank(n_blocks: int, world: int, rank: int) -> tuple[int, int]:
    return stage_intervals(n_blocks, world)[rank]

"""Work partitioning across GPUs (one process per GPU).

Two partitionings:

* instance sharding (configs 1/2): independent instances are split into
  contiguous blocks balanced by gram-build + step cost; all replicas of an
  instance stay on one GPU (they share its gram).  No data-path collective.
* tile sharding (config 4 on the fp32 symmetric path, the default for sharded
  contexts): every rank keeps the full state and streams only the upper-
  triangle gram tiles of its super-rows (tile_shard); the per-rank partial
  products G w are all-reduced once per step / sweep and every rank runs the
  same update -- one collective, no all-gather, no reconciliation;
* row sharding (fp64 / CUDA-core contexts): one instance too large for a GPU;
  rank k owns the gram rows [r0, r1) (whole row blocks of the contraction
  tile) and the state of those spins; after every Euler step (and every Jacobi
  sweep) the contraction input w is all-gathered so each rank holds the full
  vector.

These helpers are pure host logic (tests/test_dist.py drives them with
world_size 2 over gloo); the CUDA path consumes the plans.
"""
from __future__ import annotations

from typing import Sequence

ROW_QUANTUM = 128  # rows of one contraction tile (MMA M)


def instance_shard(costs: Sequence[float], world: int, rank: int) -> range:
    """Contiguous block of instance indices for `rank`, balancing sum(cost)."""
    n = len(costs)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    total = float(sum(costs))
    bounds = [0]
    acc, k = 0.0, 0
    for r in range(1, world):
        target = total * r / world
        while k < n and acc + costs[k] / 2 < target:
            acc += costs[k]
            k += 1
        bounds.append(k)
    bounds.append(n)
    return range(bounds[rank], bounds[rank + 1])


def instance_cost(N: int, M: int, n_steps: int, alternations: int) -> float:
    """Relative cost of one instance: gram build (2 N^2 M flops at ~1/8 the
    streaming rate) + the streamed gram bytes of all steps and sweeps."""
    return 2.0 * N * N * M / 8.0 + 4.0 * N * N * n_steps * alternations


def row_shard(N: int, world: int, rank: int, quantum: int = ROW_QUANTUM) -> tuple[int, int]:
    """[r0, r1) spin rows owned by `rank`: equal multiples of `quantum`
    (the last rank may hold fewer real rows; padding rows are zero)."""
    per = -(-N // (world * quantum)) * quantum
    r0 = min(N, rank * per)
    r1 = min(N, r0 + per)
    return r0, r1


def padded_rows(N: int, world: int, quantum: int = ROW_QUANTUM) -> int:
    """Global padded length so every rank's slice has the same size (all-gather)."""
    return -(-N // (world * quantum)) * quantum * world


def tile_shard(nRB: int, world: int, rank: int) -> tuple[int, int]:
    """Super-rows [P0, P1) of the symmetric gram (4 row blocks of 128 each)
    streamed by `rank`: the C runtime's own partition (cimcs_tile_shard),
    contiguous and balanced by upper-triangle tile count."""
    import ctypes as C
    from ._lib import load
    from .cimcs import _check
    a, b = C.c_int32(), C.c_int32()
    _check(load().cimcs_tile_shard(nRB, world, rank, C.byref(a), C.byref(b)))
    return a.value, b.value

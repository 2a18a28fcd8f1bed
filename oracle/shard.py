"""Oracle: KV-head sharding and the head all-gather.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper runs Qwen-7B with tensor parallelism 2 through vLLM (P:319
"vLLM's efficient tensor parallelism").  Attention is independent per KV
head, so rank r of G owns kv heads [r*Hkv/G, (r+1)*Hkv/G) and their query
heads [r*Hq/G, (r+1)*Hq/G) (GQA groups stay whole, R7).  The all-gather of
head-major outputs O [Hq/G][T][d] is a concatenation along the head axis.
"""
from __future__ import annotations

import numpy as np


def head_ranges(world: int, rank: int, num_q_heads: int, num_kv_heads: int):
    if num_kv_heads % world or num_q_heads % world:
        raise ValueError("heads must divide evenly across ranks")
    hk = num_kv_heads // world
    hq = num_q_heads // world
    return (rank * hq, (rank + 1) * hq), (rank * hk, (rank + 1) * hk)


def allgather_heads(slices):
    """Rank-ordered concatenation of [Hq/G][T][...] slices along axis 0."""
    return np.concatenate(slices, axis=0)

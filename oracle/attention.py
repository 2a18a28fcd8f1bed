"""Oracle: hybrid-batch attention over the paged KV cache.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper never writes the attention down; it delegates it to vLLM
PagedAttention and Sarathi chunked prefills (§3.6; §2.1
"Chunked prefills split a prefill request into equal-sized chunks ... without
pausing ongoing decodes"; P:205 ⑤ the mixed batch).  Hybrid batching changes
WHICH rows run together, never WHAT each row computes, so the oracle is the
plain definition (readings R1, R7, R10, R11):

  for batch row r with `visible` keys and q head h, kv head kh = h // (Hq/Hkv):
      s_t   = scale * <q_{r,h}, K_{kh}[t]>          t in [0, visible)
      m     = max_t s_t ;  p_t = exp(s_t - m) ;  l = sum_t p_t
      O[h][r]   = sum_t p_t V_{kh}[t] / l
      LSE[h][r] = m + ln l                           (natural log, R11)

with scale = 1/sqrt(d) unless overridden.  Everything is float64.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np


def to_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    """Stored representation -> float64 (bf16 bits are the top half of an fp32)."""
    if dtype == "bf16":
        return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def softmax_attend(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float) -> Tuple[np.ndarray, np.ndarray]:
    """q [g][d], k [n][d], v [n][d] (fp64) -> (o [g][d], lse [g]).  n >= 1."""
    s = (q @ k.T) * scale                      # [g][n]
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(axis=1, keepdims=True)
    o = (p @ v) / l
    lse = (m + np.log(l))[:, 0]
    return o, lse


def hybrid_attention(pool, layer: int, plan, q: np.ndarray, num_q_heads: int,
                     scale: float | None = None, rows=None) -> Tuple[np.ndarray, np.ndarray]:
    """O [Hq][T][d] and LSE [Hq][T] (float64) for every batch row of `plan`.

    `rows` optionally restricts the computation to a subset of row indices
    (other entries are NaN) so that full-size workloads can be checked on
    sampled outputs one by one."""
    Hq, Hkv, d = num_q_heads, pool.H, pool.d
    g = Hq // Hkv
    if scale is None or scale <= 0:
        scale = 1.0 / math.sqrt(d)
    T = len(plan.rows)
    O = np.full((Hq, T, d), np.nan)
    LSE = np.full((Hq, T), np.nan)
    qf = to_f64(q, pool.dtype) if q.dtype != np.float64 else q
    cache = {}
    sel = range(T) if rows is None else rows
    for r in sel:
        seq, _pos, n = plan.rows[r]
        if seq not in cache:
            kk, vv = pool.gather(layer, seq, pool.length[seq])
            cache = {seq: (to_f64(kk, pool.dtype), to_f64(vv, pool.dtype))}
        K, V = cache[seq]
        for kh in range(Hkv):
            o, lse = softmax_attend(qf[r, kh * g:(kh + 1) * g, :], K[:n, kh, :], V[:n, kh, :], scale)
            O[kh * g:(kh + 1) * g, r, :] = o
            LSE[kh * g:(kh + 1) * g, r] = lse
    return O, LSE


# ---------------------------------------------------------------------------
# a5/a6: split-KV partials and their log-sum-exp merge
# ---------------------------------------------------------------------------

def split_partial(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float):
    """Partial over one key range: (m_s, l_s, o~_s) with o~_s normalised within the split
    (m = max logit, l = sum e^{s-m}, o~ = sum e^{s-m} v / l)."""
    s = (q @ k.T) * scale
    m = s.max(axis=1)
    p = np.exp(s - m[:, None])
    l = p.sum(axis=1)
    return m, l, (p @ v) / l[:, None]


def merge_partials(parts):
    """m = max_s m_s; l = sum_s e^{m_s-m} l_s;
    o = sum_s e^{m_s-m} l_s o~_s / l; lse = m + ln l.  Parts are merged in list order."""
    ms = np.stack([p[0] for p in parts])        # [S][g]
    ls = np.stack([p[1] for p in parts])
    os_ = np.stack([p[2] for p in parts])       # [S][g][d]
    m = ms.max(axis=0)
    w = np.exp(ms - m[None, :]) * ls            # [S][g]
    l = w.sum(axis=0)
    o = (w[:, :, None] * os_).sum(axis=0) / l[:, None]
    return o, m + np.log(l)

"""Oracle: iteration-time predictor for one hybrid-batch attention launch.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's predictor maps a batch composition to latency (P:205 step ④ "A
lightweight predictor is then used to estimate the latency of the batch";
P:319 a random forest on Vidur profiles; P:744 draft: a profile lookup
table).  Its features are never published.  The north_star replaces it with
`niyama_predict_iter_time`, fitted from MEASURED kernel latency against chunk
size and decode count.  DESIGN.md reading R16 fixes the model:

  features of a batch on a shape (local heads Hq, Hkv, head dim d, element
  size e; SURVEY §8(d) "algorithmic work"):
    phi0 = 1
    phi1 = c          total prefill rows (sum of slice lengths)
    phi2 = D          decode rows
    phi3 = B_KV       = [sum_slices (o + c) + sum_decodes ctx] * Hkv * d * 2 * e   bytes
    phi4 = F          = 4 * d * Hq * [sum_slices (c*o + c(c+1)/2) + sum ctx]      flops
    phi5 = roof       = max(F / F_PEAK, B_KV / B_PEAK)                             seconds
  t_hat = theta . phi with theta >= 0, fitted by non-negative least squares on
  RELATIVE residuals (rows scaled by 1/t_meas).  theta >= 0 makes t_hat
  non-decreasing in c, D and every ctx (SPEC S:136 monotonicity).

  SPEC's affine cost model (c0 + c1*(tokens) + c2*sum ctx) is the
  special case theta = (c0, c1, c1, c2/(Hkv*d*2*e), 0, 0) on batches without a
  prefill offset; its worked examples pin eval and max_feasible_chunk.

max_feasible_chunk: the largest C in [0, min(max_chunk, remaining)]
whose batch (C prefill rows at `offset` + the decodes) predicts <= slack,
with the R18 boundary rule (<= slack within 1e-12 relative); if C = 0 is
already infeasible return (0, infeasible=True).  The oracle scans every C.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np
from scipy.optimize import nnls

F_PEAK = {"bf16": 2.25e15, "f32": 1.125e15}   # dense tensor peak, FLOP/s (B200 nominal)
B_PEAK = 8.0e12                               # HBM3e, B/s (B200 nominal)
NFEAT = 6


@dataclass
class PredShape:
    num_q_heads: int      # local (per rank)
    num_kv_heads: int     # local (per rank)
    head_dim: int
    elt_bytes: int
    dtype: str = "bf16"


@dataclass
class Sample:
    chunk_len: int        # prefill rows (single slice)
    chunk_offset: int
    num_decode: int
    sum_ctx: int          # sum of decode ctx
    seconds: float


def features(shape: PredShape, slices: Sequence[Tuple[int, int]], decode_ctx: Sequence[int]) -> np.ndarray:
    """phi for one batch; slices = [(offset, len)], decode_ctx = [ctx]."""
    slices = [(o, n) for o, n in slices if n > 0]   # a zero-length slice is no slice
    c = sum(n for _, n in slices)
    D = len(decode_ctx)
    sum_ctx = sum(decode_ctx)
    tok = sum(o + n for o, n in slices) + sum_ctx
    pairs = sum(n * o + n * (n + 1) // 2 for o, n in slices) + sum_ctx
    B = float(tok) * shape.num_kv_heads * shape.head_dim * 2 * shape.elt_bytes
    F = 4.0 * shape.head_dim * shape.num_q_heads * float(pairs)
    roof = max(F / F_PEAK[shape.dtype], B / B_PEAK)
    return np.array([1.0, float(c), float(D), B, F, roof])


def features_sample(shape: PredShape, s: Sample) -> np.ndarray:
    """Sample form: one slice (offset, len) and decodes summarised by (D, sum ctx)."""
    c, o, D, L = s.chunk_len, s.chunk_offset, s.num_decode, s.sum_ctx
    tok = (o + c if c > 0 else 0) + L
    pairs = (c * o + c * (c + 1) // 2 if c > 0 else 0) + L
    B = float(tok) * shape.num_kv_heads * shape.head_dim * 2 * shape.elt_bytes
    F = 4.0 * shape.head_dim * shape.num_q_heads * float(pairs)
    roof = max(F / F_PEAK[shape.dtype], B / B_PEAK)
    return np.array([1.0, float(c), float(D), B, F, roof])


def fit(shape: PredShape, samples: List[Sample]) -> np.ndarray:
    """theta >= 0 minimising sum ((theta.phi_i - t_i) / t_i)^2 (NNLS; columns rescaled
    to unit max for conditioning, which leaves the NNLS minimiser unchanged)."""
    if len(samples) == 0:
        raise ValueError("no samples")
    A = np.stack([features_sample(shape, s) for s in samples])
    t = np.array([s.seconds for s in samples])
    if np.any(t <= 0):
        raise ValueError("non-positive sample time")
    A = A / t[:, None]
    b = np.ones_like(t)
    colmax = np.abs(A).max(axis=0)
    colmax[colmax == 0] = 1.0
    z, _ = nnls(A / colmax, b)
    return z / colmax


def predict(theta: np.ndarray, phi: np.ndarray) -> float:
    return float(theta @ phi)


def feasible(t: float, slack: float) -> bool:
    """R18: exactly-at-deadline is a pass; 1e-12 relative guard for rounding."""
    return t <= slack + 1e-12 * max(1.0, abs(slack))


def max_feasible_chunk(theta: np.ndarray, shape: PredShape, decode_ctx: Sequence[int], offset: int,
                       remaining: int, slack: float, max_chunk: int) -> Tuple[int, bool]:
    """Brute force over every C (S:116 'largest C in [0, max_chunk] ...')."""
    cap = max(0, min(max_chunk, remaining))
    if not feasible(predict(theta, features(shape, [(offset, 0)], decode_ctx)), slack):
        return 0, True
    best = 0
    for C in range(1, cap + 1):
        if feasible(predict(theta, features(shape, [(offset, C)], decode_ctx)), slack):
            best = C
    return best, False

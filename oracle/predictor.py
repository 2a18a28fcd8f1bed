"""Oracle: iteration-time predictor for one hybrid-batch attention launch.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's predictor maps a batch composition to latency (P:205 step ④ "A
lightweight predictor is then used to estimate the latency of the batch";
P:319 a random forest on Vidur profiles; P:744 draft: a profile lookup
table).  Its features are never published.  The north_star replaces it with
`niyama_predict_iter_time`, fitted from MEASURED launch latency against chunk
size and decode count.  DESIGN.md reading R16 and section "a8 schedule model"
fix the model, written out here step by step:

  shape: local heads Hq, Hkv, head dim d, element bytes e; g = Hq/Hkv,
  R = max(1, 128 // g) chunk rows per prefill tile; NSM = 148 SMs.
  1. tile queue: prefill slices (o, c > 0) sorted by o + c descending
     (stable); per slice q tiles qt = nqt-1 .. 0 (nqt = ceil(c/R)), each
     repeated Hkv times, cost = ceil((o + min(c, (qt+1) R)) / 128) + SETUP.
  2. decode units: split_len q = the smallest power of two s >= 128 with
     2 s^2 >= raw^2 (s >= raw / sqrt 2: the power of two nearest raw in log
     scale), raw = ceil(max(1, sumL*Hkv) / (4*NSM*8)), and ceil(max_ctx/s) <=
     4095 (capped at 2^20); a row of ctx L is n_f = ceil(L/q) - 1 pieces of q keys
     plus its last L - n_f*q keys in pieces of min(q, max(256, q // TAIL_DIV));
     units = Hkv * sum over rows of the piece count.
  3. grid = max(1, min(NSM, tiles + ceil(units/8))); prefill CTAs n_p = 0
     without tiles, = grid without units, else ceil(grid*wp/(wp+wd)) with
     wp = (sum of tile costs) * STEP_BYTES and wd = sumL*Hkv*d*2*e (times
     WIDE_GROUP_DECODE_WEIGHT when g = Hq/Hkv > 4), raised to
     min(ceil(tiles/4), ceil(grid/2)), then capped at tiles and at grid, and at
     least 1.
  4. list scheduling: each tile in queue order goes to the prefill CTA that
     frees first; f_1 <= ... <= f_np the finish times (in steps).
  5. fluid decode: B_d = sumL*Hkv*d*2*e bytes stream at min(BW, k*r_cta),
     k = grid - (prefill CTAs still busy); a step lasts tau seconds.
     T_p = tau * f_np; T_d = the time B_d is done (0 when B_d = 0).
  6. phi = [1, c + D, D, sumL, max(T_d, T_p), min(T_d, T_p)];
     t_hat = theta[0:6] . phi with theta[0:6] >= 0; theta[6:9] = (tau, r_cta, BW).

  SPEC's affine cost model (c0 + c1*(tokens) + c2*sum ctx) is the
  special case theta[0:6] = (c0, c1, 0, c2, 0, 0); its worked examples pin
  eval and max_feasible_chunk.

fit (R16): for every (tau, r_cta, BW) of a grid (tau-major, then r_cta, then
BW; values lo + i*step, i = 0..round((hi-lo)/step)), theta[0:6] by
non-negative least squares of phi_i/t_i against 1 (columns scaled to unit
max); the grid point with the least sum of squared relative residuals wins
(the first within 1e-9 relative of the minimum).  A sample (c, o, D, sumL)
stands for the batch {slice (o, c) if c > 0} + D decodes with sumL spread
evenly (the first sumL mod D of them one longer).

max_feasible_chunk: C = 0 infeasible -> (0, infeasible);
cap feasible -> cap; else bisection lo = 0, hi = cap, mid = (lo+hi)//2 until
hi = lo + 1, returning lo, so t(C) <= slack < t(C+1).  When t_hat is
non-decreasing in C this is S:119's "largest C", which
`largest_feasible_chunk` computes by scanning every C.
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np
from scipy.optimize import nnls

NSM = 148
TAIL_DIV = 4
STEP_BYTES = 160e3
WIDE_GROUP_DECODE_WEIGHT = 1.8   # include/niyama.h NIYAMA_WIDE_GROUP_DECODE_WEIGHT
SETUP = 2
NFEAT = 6
NPARAM = 9
DEFAULT_GRID = (0.5e-6, 2.5e-6, 0.1e-6, 30e9, 120e9, 5e9, 5.0e12, 8.4e12, 0.2e12)


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


@dataclass
class Sched:
    rows: int
    D: int
    sum_ctx: int
    Bd: float
    grid: int
    np_: int
    fin: List[int] = field(default_factory=list)
    units: int = 0


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def split_len(sum_ctx: int, max_ctx: int, hkv: int, nsm: int = NSM) -> int:
    """Step 2: decode split length."""
    raw = cdiv(max(1, sum_ctx * hkv), 4 * nsm * 8)
    s = 128
    while (2 * s * s < raw * raw or cdiv(max_ctx, s) > 4095) and s < (1 << 20):
        s *= 2
    return s


def tile_queue(shape: PredShape, slices: Sequence[Tuple[int, int]]) -> List[int]:
    """Step 1: tile costs in queue order."""
    g = shape.num_q_heads // shape.num_kv_heads
    R = max(1, 128 // g)
    live = [(o, c) for o, c in slices if c > 0]
    live = sorted(live, key=lambda sc: -(sc[0] + sc[1]))         # Python's sort is stable
    costs = []
    for o, c in live:
        for qt in range(cdiv(c, R) - 1, -1, -1):
            cost = cdiv(o + min(c, (qt + 1) * R), 128) + SETUP
            costs += [cost] * shape.num_kv_heads
    return costs


def cta_split(n_tiles: int, n_units: int, tile_cost: int, sum_ctx: int, shape: PredShape) -> Tuple[int, int]:
    """Step 3: (grid, prefill CTAs)."""
    grid = max(1, min(NSM, n_tiles + cdiv(n_units, 8)))
    if n_tiles == 0:
        return grid, 0
    if n_units == 0:
        return grid, grid
    wp = float(tile_cost) * STEP_BYTES
    wd = float(sum_ctx) * shape.num_kv_heads * shape.head_dim * 2.0 * shape.elt_bytes
    if shape.num_q_heads // shape.num_kv_heads > 4:   # 8 decode warps per CTA instead of 12
        wd *= WIDE_GROUP_DECODE_WEIGHT
    n_p = math.ceil(grid * wp / (wp + wd))
    n_p = max(n_p, min(cdiv(n_tiles, 4), cdiv(grid, 2)))
    n_p = min(n_p, n_tiles, grid)
    return grid, max(1, n_p)


def list_schedule(costs: Sequence[int], m: int) -> List[int]:
    """Step 4: finish times of m machines when each job in order goes to the earliest-free one."""
    if not costs:
        return []
    heap = [0] * m
    for c in costs:
        t = heapq.heappop(heap)
        heapq.heappush(heap, t + c)
    return sorted(heap)


def schedule(shape: PredShape, slices: Sequence[Tuple[int, int]], decode_ctx: Sequence[int]) -> Sched:
    costs = tile_queue(shape, slices)
    D = len(decode_ctx)
    L = int(sum(decode_ctx))
    units = 0
    if D:
        q = split_len(L, int(max(decode_ctx)), shape.num_kv_heads)
        small = min(q, max(256, q // TAIL_DIV))
        for x in decode_ctx:
            nf = cdiv(int(x), q) - 1
            units += (nf + cdiv(int(x) - nf * q, small)) * shape.num_kv_heads
    grid, n_p = cta_split(len(costs), units, sum(costs), L, shape)
    Bd = float(L) * shape.num_kv_heads * shape.head_dim * 2.0 * shape.elt_bytes
    rows = sum(c for _, c in slices if c > 0)
    return Sched(rows, D, L, Bd, grid, n_p, list_schedule(costs, n_p), units)


def phi(s: Sched, tau: float, rc: float, bw: float) -> np.ndarray:
    """Step 5-6."""
    Tp = tau * float(s.fin[-1]) if s.fin else 0.0
    Td = 0.0
    if s.Bd > 0:
        t, done, busy = 0.0, 0.0, s.np_
        for f in s.fin:
            tf = tau * float(f)
            rate = min(bw, (s.grid - busy) * rc)
            if rate > 0 and done + rate * (tf - t) >= s.Bd:
                Td = t + (s.Bd - done) / rate
                break
            done += rate * (tf - t)
            t = tf
            busy -= 1
        else:
            Td = t + (s.Bd - done) / min(bw, s.grid * rc)
    return np.array([1.0, float(s.rows + s.D), float(s.D), float(s.sum_ctx), max(Td, Tp), min(Td, Tp)])


def predict(theta, shape: PredShape, slices: Sequence[Tuple[int, int]], decode_ctx: Sequence[int]) -> float:
    theta = np.asarray(theta, dtype=float)
    return float(np.dot(theta[:NFEAT], phi(schedule(shape, slices, decode_ctx), *theta[NFEAT:])))


def sample_batch(s: Sample) -> Tuple[List[Tuple[int, int]], List[int]]:
    slices = [(s.chunk_offset, s.chunk_len)] if s.chunk_len > 0 else []
    ctx = []
    if s.num_decode:
        base, rem = divmod(s.sum_ctx, s.num_decode)
        ctx = [base + (1 if j < rem else 0) for j in range(s.num_decode)]
    return slices, ctx


def grid_values(lo: float, hi: float, step: float) -> List[float]:
    n = int(math.floor((hi - lo) / step + 0.5)) + 1
    return [lo + float(i) * step for i in range(n)]


def fit(shape: PredShape, samples: List[Sample], grid=DEFAULT_GRID) -> np.ndarray:
    if len(samples) == 0:
        raise ValueError("no samples")
    t = np.array([s.seconds for s in samples], dtype=float)
    if np.any(t <= 0):
        raise ValueError("non-positive sample time")
    scheds = [schedule(shape, *sample_batch(s)) for s in samples]
    cands = []
    for tau in grid_values(*grid[0:3]):
        for rc in grid_values(*grid[3:6]):
            for bw in grid_values(*grid[6:9]):
                Phi = np.stack([phi(sc, tau, rc, bw) for sc in scheds])
                A = Phi / t[:, None]
                colmax = np.abs(A).max(axis=0)
                colmax[colmax == 0] = 1.0
                z, _ = nnls(A / colmax, np.ones_like(t))
                lin = z / colmax
                score = float(np.sum((Phi @ lin / t - 1.0) ** 2))
                cands.append((score, np.concatenate([lin, [tau, rc, bw]])))
    best = min(c[0] for c in cands)
    for score, theta in cands:
        if score <= best * (1.0 + 1e-9):
            return theta
    raise AssertionError("unreachable")


def feasible(t: float, slack: float) -> bool:
    """R18: exactly-at-deadline is a pass; 1e-12 relative guard for rounding."""
    return t <= slack + 1e-12 * max(1.0, abs(slack))


def max_feasible_chunk(theta, shape: PredShape, decode_ctx: Sequence[int], offset: int, remaining: int,
                       slack: float, max_chunk: int) -> Tuple[int, bool]:
    """S:137 boundary by bisection (module docstring)."""
    def t_of(C):
        return predict(theta, shape, [(offset, C)], decode_ctx)
    cap = max(0, min(max_chunk, remaining))
    if not feasible(t_of(0), slack):
        return 0, True
    if feasible(t_of(cap), slack):
        return cap, False
    lo, hi = 0, cap
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if feasible(t_of(mid), slack):
            lo = mid
        else:
            hi = mid
    return lo, False


def largest_feasible_chunk(theta, shape: PredShape, decode_ctx: Sequence[int], offset: int, remaining: int,
                           slack: float, max_chunk: int) -> Tuple[int, bool]:
    """S:119 literally: the largest C in [0, cap] whose batch is feasible (scan)."""
    cap = max(0, min(max_chunk, remaining))
    if not feasible(predict(theta, shape, [(offset, 0)], decode_ctx), slack):
        return 0, True
    best = 0
    for C in range(1, cap + 1):
        if feasible(predict(theta, shape, [(offset, C)], decode_ctx), slack):
            best = C
    return best, False

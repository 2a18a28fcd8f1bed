"""Oracle: the a8 iteration-time predictor and the a1 chunk choice.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's predictor maps a batch composition to latency (P:205 step ④ "A
lightweight predictor is then used to estimate the latency of the batch";
P:319 a random forest on Vidur profiles; P:744 draft: a profile lookup table).
Its features are never published; the north_star asks for
`niyama_predict_iter_time` "fitted from measured kernel latency against chunk
size and decode count".  DESIGN.md reading R16 and §6.4 fix the model: an
event model of one hybrid-attention launch, written out here step by step.

Inputs.  The batch (prefill slices (o, c), decode contexts) defines the WORK —
the causal key range of every prefill q tile and the key pieces of every decode
row — and the launch configuration (`Launch`: split length q, small-piece
length, grid, prefill CTAs n_p, decode warps per CTA) is the kernel's plan
(`niyama_plan_info`), an input here: the oracle models "this launch", it does
not re-derive the planner's heuristics.

  shape: local heads Hq, Hkv, head dim d, element bytes e; g = Hq / Hkv,
  R = 128 // g chunk rows per prefill tile; NSM = 148.
  1. tile queue: slices sorted by o + c descending (stable); per slice the q tiles
     qt = nqt-1 .. 0 (nqt = ceil(c / R)), each Hkv times, with
     nk = ceil((o + min(c, (qt+1) R)) / 128) key steps (the keys row o + (qt+1) R - 1
     sees, causal), cut into P split-K parts of floor((i+1) nk/P) - floor(i nk/P)
     steps (P from the plan's target, a launch input).
  2. unit queue: rows by ctx descending; a row of L keys has n_f = ceil(L/q) - 1
     full pieces of q keys (each Hkv units, row by row), then the remaining
     L - n_f q keys of every row in pieces of `small` keys, all those pieces
     longest first (each Hkv units).  A unit of k keys streams k d 2 e bytes.
  3. event model, two clocks.  Prefill CTAs advance together on a step clock S
     at 1/tau(t) steps/s, tau = tau0 + tau_p P/NSM + tau_d B/W (P prefill CTAs
     busy, B decode warps busy, W = grid x warps per CTA); the queue's next tile
     goes to a free prefill CTA; a tile of s steps taken at S = x ends at
     S = x + s + sigma, except a CTA's first tile, which ends at S = s + sigma0
     (its setup includes the CTA's start).  Decode warps advance together on a byte clock V at
     rate = min(r_w, BW / B, r_cta (grid - P) / B) / (1 + gamma P / NSM) bytes/s
     each; a free warp takes the queue's next unit; a unit of b bytes taken at
     V = v ends at V = v + b + u0 r_w.  The grid - n_p decode CTAs' warps are free
     at t = 0, a prefill CTA's warps when it finds the tile queue empty.  The next
     event is the earlier of the first tile end and the first unit end.
     T_sim = the time the last tile or unit ends.
  4. t_hat = th[0] + th[1] (rows + D) + th[2] D + th[3] sum ctx + th[4] units
             + th[5] T_sim,
     th[6:16] = (tau0, tau_p, tau_d, sigma, r_w, u0, BW, gamma, r_cta, sigma0).

  SPEC's affine cost model (c0 + c1 * tokens + c2 * sum ctx) is the
  special case th[0:6] = (c0, c1, 0, c2, 0, 0); its worked examples pin eval and
  max_feasible_chunk.

fit (R16): th[6:16] minimise the sum of squared relative errors, th[0:5] >= 0 by
non-negative least squares on relative residuals at fixed th[5] = 1 (the
library runs Nelder-Mead on the logarithms; any minimiser may be used here).

max_feasible_chunk: C = 0 infeasible -> (0, infeasible);
cap feasible -> cap; else bisection lo = 0, hi = cap, mid = (lo+hi)//2 until
hi = lo + 1, returning lo, so t(C) <= slack < t(C+1).  When t_hat is
non-decreasing in C this is S:119's "largest C", which
`largest_feasible_chunk` computes by scanning every C.
"""
from __future__ import annotations

import bisect
import math
from dataclasses import dataclass, field
from typing import Callable, List, Sequence, Tuple

import numpy as np
from scipy.optimize import nnls

NSM = 148
NPARAM = 16
NLIN = 6


@dataclass
class PredShape:
    num_q_heads: int      # local (per rank)
    num_kv_heads: int     # local (per rank)
    head_dim: int
    elt_bytes: int
    dtype: str = "bf16"


@dataclass
class Launch:
    """The launch configuration of a batch: the plan's choices (niyama_plan_info)."""

    split_len: int
    small: int            # small-piece length min(q, max(tail_min, q // tail_div))
    grid: int
    prefill_ctas: int
    warps_per_cta: int    # 12 when g <= 4, else 8


@dataclass
class Work:
    rows: int
    D: int
    sum_ctx: int
    units: int
    tiles: List[int] = field(default_factory=list)        # steps per tile, queue order
    pieces: List[float] = field(default_factory=list)     # bytes per unit, queue order


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def work(shape: PredShape, slices: Sequence[Tuple[int, int]], decode_ctx: Sequence[int], q: int, small: int,
         parts_target: int = 1) -> Work:
    """Steps 1-2.  parts_target: the plan's split-K target (a launch input); a slice's q tiles
    are cut into P = min(target, its shortest tile's steps // 4) (>= 1) key parts."""
    g = shape.num_q_heads // shape.num_kv_heads
    R = max(1, 128 // g)
    live = sorted([(o, c) for o, c in slices if c > 0], key=lambda sc: -(sc[0] + sc[1]))   # stable
    tiles = []
    for o, c in live:
        nks = [cdiv(o + min(c, (qt + 1) * R), 128) for qt in range(cdiv(c, R) - 1, -1, -1)]
        P = max(1, min(parts_target, nks[-1] // 4)) if parts_target > 1 else 1
        for nk in nks:
            for _ in range(shape.num_kv_heads):
                tiles += [(i + 1) * nk // P - i * nk // P for i in range(P)]
    bpt = float(shape.head_dim * 2 * shape.elt_bytes)
    pieces, tail, units = [], [], 0
    for L in sorted((int(x) for x in decode_ctx), reverse=True):
        nf = cdiv(L, q) - 1
        pieces += [q * bpt] * (nf * shape.num_kv_heads)
        k0 = nf * q
        while k0 < L:
            tail.append(min(L, k0 + small) - k0)
            k0 += small
        units += (nf + cdiv(L - nf * q, small)) * shape.num_kv_heads
    for k in sorted(tail, reverse=True):
        pieces += [k * bpt] * shape.num_kv_heads
    return Work(sum(c for _, c in live), len(decode_ctx), int(sum(decode_ctx)), units, tiles, pieces)


class _Clock:
    """Ascending multiset of end coordinates (one entry per machine)."""

    def __init__(self):
        self.v: List[float] = []

    def add(self, x: float):
        bisect.insort(self.v, x)


def simulate(w: Work, ln: Launch, nl: Sequence[float]) -> float:
    """Step 3: the two-clock event model; returns T_sim."""
    tau0, tau_p, tau_d, sigma, r_w, u0, bw, gamma, r_cta, sigma0 = [float(x) for x in nl]
    has_tiles = len(w.tiles) > 0 and ln.prefill_ctas > 0
    W = float(ln.grid * ln.warps_per_cta)
    cta, busy = _Clock(), _Clock()
    tq, uq = list(w.tiles), list(w.pieces)
    ti = ui = 0
    t = S = V = 0.0

    def take_units(n):
        nonlocal ui
        while n > 0 and ui < len(uq):
            busy.add(V + uq[ui] + u0 * r_w)
            ui += 1
            n -= 1

    def take_tiles(n):          # returns the CTAs that found the queue empty
        nonlocal ti
        while n > 0 and ti < len(tq):
            cta.add(S + tq[ti] + sigma)
            ti += 1
            n -= 1
        return n

    if has_tiles:
        S = sigma0 - sigma
        take_units((ln.grid - ln.prefill_ctas) * ln.warps_per_cta)
        take_units(take_tiles(ln.prefill_ctas) * ln.warps_per_cta)
        S = 0.0
    else:
        take_units(ln.grid * ln.warps_per_cta)
    while cta.v or busy.v:
        P, B = len(cta.v), len(busy.v)
        tau = tau0 + tau_p * P / NSM + tau_d * B / W
        rate = 0.0
        if B:
            rate = min(r_w, bw / B, r_cta * max(1.0, float(ln.grid - P)) / B) / (1.0 + gamma * P / NSM)
        dt_p = (cta.v[0] - S) * tau if P else math.inf
        dt_d = (busy.v[0] - V) / rate if B else math.inf
        if dt_p <= dt_d:
            t += dt_p
            if B:
                V += dt_p * rate
            S = cta.v.pop(0)
            take_units(take_tiles(1) * ln.warps_per_cta)
        else:
            t += dt_d
            if P:
                S += dt_d / tau
            V = busy.v.pop(0)
            take_units(1)
    return t


def features(w: Work, t_sim: float) -> np.ndarray:
    return np.array([1.0, float(w.rows + w.D), float(w.D), float(w.sum_ctx), float(w.units), t_sim])


def predict(theta, w: Work, ln: Launch) -> float:
    th = np.asarray(theta, dtype=float)
    return float(np.dot(th[:NLIN], features(w, simulate(w, ln, th[NLIN:]))))


def tiles_per_cta(w: Work, ln: Launch) -> List[int]:
    """Tiles each prefill CTA runs under step 3's list schedule (all prefill CTAs share the
    step clock, so the assignment is the list schedule of (s + sigma) costs; sigma and
    sigma0 shift every CTA alike and do not change it)."""
    if not w.tiles or ln.prefill_ctas == 0:
        return []
    free = [(0.0, c) for c in range(ln.prefill_ctas)]
    count = [0] * ln.prefill_ctas
    for s in w.tiles:
        free.sort()
        t, c = free.pop(0)
        count[c] += 1
        free.append((t + s, c))
    return count


def fit_linear(ws: Sequence[Work], lns: Sequence[Launch], t: np.ndarray, nl) -> Tuple[np.ndarray, float]:
    """th[0:5] >= 0 by NNLS on relative residuals with th[5] = 1 (module docstring)."""
    Ts = np.array([simulate(w, ln, nl) for w, ln in zip(ws, lns)])
    F = np.array([features(w, x)[:5] for w, x in zip(ws, Ts)])
    A = F / t[:, None]
    cm = np.abs(A).max(axis=0)
    cm[cm == 0] = 1.0
    z, _ = nnls(A / cm, 1.0 - Ts / t)
    lin = np.concatenate([z / cm, [1.0]])
    err = (F @ lin[:5] + Ts) / t - 1.0
    return lin, float(np.sum(err ** 2))


def fit(ws, lns, t, minimiser: Callable, start) -> np.ndarray:
    """Step 'fit': minimiser(objective, x0) -> x over log(th[6:16])."""
    t = np.asarray(t, dtype=float)
    x = minimiser(lambda x: fit_linear(ws, lns, t, np.exp(x))[1], np.log(np.asarray(start, dtype=float)))
    nl = np.exp(x)
    lin, _ = fit_linear(ws, lns, t, nl)
    return np.concatenate([lin, nl])


def feasible(t: float, slack: float) -> bool:
    """R18: exactly-at-deadline is a pass; 1e-12 relative guard for rounding."""
    return t <= slack + 1e-12 * max(1.0, abs(slack))


def max_feasible_chunk(t_of: Callable[[int], float], remaining: int, slack: float, max_chunk: int) -> Tuple[int, bool]:
    """S:137 boundary by bisection (module docstring); t_of(C) = t_hat of the batch with C rows."""
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


def largest_feasible_chunk(t_of: Callable[[int], float], remaining: int, slack: float,
                           max_chunk: int) -> Tuple[int, bool]:
    """S:119 literally: the largest C in [0, cap] whose batch is feasible (scan)."""
    cap = max(0, min(max_chunk, remaining))
    if not feasible(t_of(0), slack):
        return 0, True
    best = 0
    for C in range(1, cap + 1):
        if feasible(t_of(C), slack):
            best = C
    return best, False


def affine(c0: float, c1: float, c2: float, slices, decode_ctx) -> float:
    """SPEC S:107-115 written out: c0 + c1 * (prefill tokens + decodes) + c2 * sum ctx."""
    return c0 + c1 * (sum(c for _, c in slices) + len(decode_ctx)) + c2 * float(sum(decode_ctx))

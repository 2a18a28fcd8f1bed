"""Oracle: deadlines, slack and the per-iteration chunk choice.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3.2:
  Eq. 1  D_first = t_arrival + SLO_TTFT
  Eq. 2  D_n     = t_arrival + SLO_TTFT + (n - 1) * SLO_TBT      (n = token position, n >= 1)
  Eq. 3  D_total = t_arrival + SLO_TTLT
PAPER.md §3.3: "For each request in the decode queue, we define slack as
the difference between the deadline for the next token (eq 2) and current
time ... we calculate the maximum chunk size which can be used for the current
batch without violating any deadline."

Readings: R17 non-interactive decodes contribute the SPEC pacing
bound (D_total - now) / max(1, est_remaining_tokens); R18 a latency
exactly equal to the slack is feasible; the batch's binding slack is the
minimum over decodes, +inf with no decodes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class DecodeQoS:
    """QoS state of one running decode (mirrors `niyama_decode_qos`, include/niyama.h)."""

    interactive: bool
    t_arrival: float
    slo_ttft: float = 0.0
    slo_tbt: float = 0.0
    slo_ttlt: float = 0.0
    next_token: int = 1          # 1-based position n of the token this iteration emits (Eq. 2)
    est_remaining: int = 1       # non-interactive: estimated tokens still to decode (R17)


def deadline_first(t_arrival: float, slo_ttft: float) -> float:
    return t_arrival + slo_ttft                                   # Eq. 1


def deadline_token(t_arrival: float, slo_ttft: float, slo_tbt: float, n: int) -> float:
    if n < 1:
        raise ValueError("token position n >= 1 (Eq. 2)")
    return t_arrival + slo_ttft + (n - 1) * slo_tbt               # Eq. 2


def deadline_total(t_arrival: float, slo_ttlt: float) -> float:
    return t_arrival + slo_ttlt                                   # Eq. 3


def decode_slack(q: DecodeQoS, now: float) -> float:
    if q.interactive:
        return deadline_token(q.t_arrival, q.slo_ttft, q.slo_tbt, q.next_token) - now
    return (deadline_total(q.t_arrival, q.slo_ttlt) - now) / max(1, q.est_remaining)


def min_slack(decodes, now: float) -> float:
    s = math.inf
    for q in decodes:
        s = min(s, decode_slack(q, now))
    return s

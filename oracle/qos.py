"""Oracle: Niyama's per-replica QoS scheduler core (config 5).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, smoke() and
bench.py's cpu_baseline leg may import this module.  The product scheduler is
C++ (`niyama_sched_*`, include/niyama.h); the two share no code.

Written step by step from PAPER.md §3 (P:205 pipeline ①-⑦; Eq. 1-3;
P:246-251 dynamic chunking; P:258-287 hybrid prioritization Eq. 4-5, eager
relegation, selective preemption; P:301 multi-fill, Fig. 6) with SPEC.md's
operational rules where the paper is silent.  Readings (DESIGN.md
§2, R21-R29):

  R21 token positions: a request enters the decode queue with decoded = 0;
      its k-th decode iteration emits token n = k, so a decode's slack
      uses D_{decoded+1} (Eq. 2).
  R22 relegation order ("Only when there are no more low-priority
      requests"): every iteration, all Low-priority prefill-queue
      requests whose status != OK are relegated; High-priority ones with
      status != OK only in an iteration that relegated no Low one.
  R23 "about to violate" horizon: TTFT case deadline < now +
      Prefill_rem + decode_token_s (the first token comes from the first decode
      iteration, R21); TTLT case deadline < now + Prefill_rem + Decode_rem.
  R24 Prefill_rem (Eq. 4-5; "time to process remaining prefill tokens of
      this request alone"): sum over max_chunk-sized chunks, from the request's
      current prefill offset, of the cost model's prefill-only batch time.
  R25 Decode_rem (Eq. 5; "over-approximate it by two standard
      deviations"): max(0, mean + 2 std - decoded) tokens (Welford history per
      app, the prior before min_samples completions) x decode_token_s seconds
      per decode iteration (a scheduler setting).
  R26 selective preemption: the in-flight request is the prefill-queue
      request with 0 < prefill_done that was scheduled last; it is displaced by
      a higher-priority candidate only if its status stays OK with `now`
      advanced by the iteration's predicted latency; otherwise it goes first.
      With preemption NEVER it always goes first; ALWAYS = priority order
      alone (the EDF / SRPF baselines, "preemptive").
  R27 multi-fill (Fig. 6): the budget is max_feasible_chunk for
      the head candidate's offset; slices are filled greedily in candidate
      order; then, if the batch as filled predicts above the min slack, the
      last slice is shrunk (bisection on its length) until it fits.
  R28 relegated service (P:205 ③): only when no primary prefill
      candidate remains, the relegated queue's head (earliest original
      deadline, then arrival, then id) is the candidate; never re-promoted.
  R29 decodes of relegated requests do not bind the slack (they are counted
      violated already, "may finish late").
  R31 an interactive decode whose next-token deadline has already passed (the
      token is late whatever the chunk) binds the slack at its SLO_TBT: it is
      paced, not chased, so one late request does not starve every prefill
      (measured in the config-5 replay: chasing collapsed at 1.5x load).
  R32 KV admission (not in the paper; SPEC lists memory as a non-goal):
      with a token budget, the fill stops where the tokens held by unfinished
      requests (prefill done + decoded) plus the batch's new tokens reach it.
  R30 an iteration's time = fixed_s + layers x the cost model's time of the
      batch (the model predicts one layer's launch, a8; defaults 0 and 1).

Policies (S:262-268, P:434 baselines): NIYAMA (Eq. 4-5 key), FCFS (arrival),
EDF (TTFT / TTLT deadline), SJF (prompt tokens), SRPF (remaining prompt
tokens).  Ties break by (arrival, id).  The cost model is any object
with `iter_time(slices, decode_ctx) -> seconds` (slices = [(offset, len)]).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from oracle.sched import deadline_first, deadline_token, deadline_total

NIYAMA, FCFS, EDF, SJF, SRPF = 0, 1, 2, 3, 4
NEVER, SELECTIVE, ALWAYS = 0, 1, 2
OK, VIOLATED, WILL_VIOLATE = 0, 1, 2


@dataclass
class QoS:
    """QoS spec: Interactive -> slo_ttft, slo_tbt; NonInteractive -> slo_ttlt."""

    interactive: bool
    slo_ttft: float = 0.0
    slo_tbt: float = 0.0
    slo_ttlt: float = 0.0


@dataclass
class Config:
    policy: int = NIYAMA
    alpha: float = 0.0
    dynamic_chunk: bool = True     # P:246 dynamic chunking; False = fixed_chunk (Sarathi baselines)
    fixed_chunk: int = 256
    max_chunk: int = 2048          # P:420 "large chunk size of 2K"
    relegation: bool = True
    preemption: int = 1            # 0 never (Sarathi-FCFS), 1 selective, 2 by priority alone
    multi_fill: bool = True
    min_samples: int = 30
    prior_mean: float = 415.0      # ShareGPT decode p50 (Table 1)
    prior_std: float = 300.0
    decode_token_s: float = 0.05
    layers: float = 1.0            # an iteration = fixed_s + layers x the cost model's batch time (R30)
    fixed_s: float = 0.0
    kv_token_budget: int = 0       # R32: 0 = unlimited


@dataclass
class Req:
    id: int
    t_arrival: float
    prompt: int
    qos: QoS
    low: bool = False
    app: int = 0
    prefill_done: int = 0
    decoded: int = 0
    state: str = "prefill"        # prefill | decode | relegated | done
    relegated: bool = False
    tokens: List[float] = field(default_factory=list)


@dataclass
class Batch:
    slices: List[Tuple[int, int, int]]      # (id, offset, len)
    decodes: List[Tuple[int, int]]          # (id, ctx incl. the new token, R4)
    budget: int
    predicted: float
    min_slack: float
    infeasible: bool
    relegated: List[int]


class History:
    """Per-app decode-length history, Welford."""

    def __init__(self):
        self.n: Dict[int, int] = {}
        self.mean: Dict[int, float] = {}
        self.m2: Dict[int, float] = {}

    def add(self, app: int, x: int):
        n = self.n.get(app, 0) + 1
        mean = self.mean.get(app, 0.0)
        d = x - mean
        mean += d / n
        self.m2[app] = self.m2.get(app, 0.0) + d * (x - mean)
        self.n[app], self.mean[app] = n, mean

    def estimate(self, app: int, cfg: Config) -> float:
        """mean + 2 std, the prior before min_samples completions."""
        n = self.n.get(app, 0)
        if n < max(1, cfg.min_samples):
            return cfg.prior_mean + 2.0 * cfg.prior_std
        std = math.sqrt(self.m2[app] / n)
        return self.mean[app] + 2.0 * std


class Scheduler:
    def __init__(self, cfg: Config, model):
        self.cfg = cfg
        self.model = model
        self.reqs: Dict[int, Req] = {}
        self.hist = History()
        self.inflight: Optional[int] = None
        self.last: Optional[Batch] = None

    def iter_time(self, slices, ctx) -> float:
        """R30: one iteration runs the batch through every layer."""
        return self.cfg.fixed_s + self.cfg.layers * self.model.iter_time(slices, ctx)

    # ---- requests ----
    def submit(self, r: Req):
        if r.prompt < 1 or r.id in self.reqs:
            raise ValueError("prompt >= 1 and a new id")
        self.reqs[r.id] = r

    # ---- Eq. 1-5 ----
    def prefill_rem(self, r: Req) -> float:
        """R24."""
        t, off = 0.0, r.prefill_done
        while off < r.prompt:
            c = min(self.cfg.max_chunk, r.prompt - off)
            t += self.iter_time([(off, c)], [])
            off += c
        return t

    def decode_rem(self, r: Req) -> float:
        """R25."""
        est = max(0.0, self.hist.estimate(r.app, self.cfg) - r.decoded)
        return est * self.cfg.decode_token_s

    def deadline(self, r: Req) -> float:
        if r.qos.interactive:
            return deadline_first(r.t_arrival, r.qos.slo_ttft)          # Eq. 1
        return deadline_total(r.t_arrival, r.qos.slo_ttlt)             # Eq. 3

    def priority(self, r: Req) -> Tuple[float, float, int]:
        c = self.cfg
        if c.policy == FCFS:
            v = r.t_arrival
        elif c.policy == EDF:
            v = self.deadline(r)
        elif c.policy == SJF:
            v = float(r.prompt)
        elif c.policy == SRPF:
            v = float(r.prompt - r.prefill_done)
        else:
            work = self.prefill_rem(r)
            if not r.qos.interactive:
                work += self.decode_rem(r)                              # Eq. 5
            v = self.deadline(r) + c.alpha * work                       # Eq. 4
        return (v, r.t_arrival, r.id)

    def status(self, r: Req, now: float) -> int:
        """Violation checker (P:205 ②; R23)."""
        d = self.deadline(r)
        if d < now:
            return VIOLATED
        horizon = self.prefill_rem(r)
        if not r.qos.interactive:
            horizon += self.decode_rem(r)
        else:
            horizon += self.cfg.decode_token_s      # R23: the first token needs one decode iteration (R21)
        return WILL_VIOLATE if d < now + horizon else OK

    # ---- slack (oracle.sched) ----
    def decode_slack(self, r: Req, now: float) -> float:
        if r.qos.interactive:
            s = deadline_token(r.t_arrival, r.qos.slo_ttft, r.qos.slo_tbt, r.decoded + 1) - now      # R21
            return s if s >= 0.0 else r.qos.slo_tbt                                                   # R31
        est = max(1.0, self.hist.estimate(r.app, self.cfg) - r.decoded)
        return (deadline_total(r.t_arrival, r.qos.slo_ttlt) - now) / est                        # R17

    # ---- one iteration (P:205 ①-⑤) ----
    def next_batch(self, now: float) -> Batch:
        c = self.cfg
        if self.last is not None and (self.last.slices or self.last.decodes):
            raise ValueError("complete() the outstanding batch first")
        decodes = sorted((r for r in self.reqs.values() if r.state == "decode"), key=lambda r: (r.t_arrival, r.id))
        dec = [(r.id, r.prompt + r.decoded + 1) for r in decodes]
        ctx = [x for _, x in dec]
        slack = math.inf
        for r in decodes:
            if not r.relegated:                                         # R29
                slack = min(slack, self.decode_slack(r, now))

        # ① order the prefill queue, ②-③ relegate violators (R22)
        queue = sorted((r for r in self.reqs.values() if r.state == "prefill"), key=self.priority)
        relegated: List[int] = []
        if c.relegation:
            st = {r.id: self.status(r, now) for r in queue}
            low = [r for r in queue if r.low and st[r.id] != OK]
            chosen = low if low else [r for r in queue if not r.low and st[r.id] != OK]
            for r in chosen:
                r.state, r.relegated = "relegated", True
                relegated.append(r.id)
            queue = [r for r in queue if r.state == "prefill"]
        if not queue:                                                   # R28
            rq = sorted((r for r in self.reqs.values() if r.state == "relegated"),
                        key=lambda r: (self.deadline(r), r.t_arrival, r.id))
            queue = rq[:1] if not c.multi_fill else rq

        # selective preemption (R26)
        if self.inflight is not None and queue and queue[0].id != self.inflight and c.preemption != ALWAYS:
            cur = self.reqs.get(self.inflight)
            if cur is not None and cur in queue and 0 < cur.prefill_done:
                keep = True
                if c.preemption == SELECTIVE:
                    head = queue[0]
                    delay = self.iter_time([(head.prefill_done, min(c.max_chunk, head.prompt - head.prefill_done))], ctx)
                    keep = self.status(cur, now + delay) != OK
                if keep:
                    queue = [cur] + [r for r in queue if r is not cur]

        # ④ chunk budget
        infeasible = False
        if not queue:
            budget = 0
        elif not c.dynamic_chunk:
            budget = c.fixed_chunk
        else:
            head = queue[0]
            budget, infeasible = self.max_chunk(ctx, head.prefill_done, slack, c.max_chunk)

        # ⑤ fill (R27), within the KV token budget (R32)
        slices: List[Tuple[int, int, int]] = []
        left = budget
        if c.kv_token_budget > 0:
            held = len(dec) + sum(r.prefill_done + r.decoded for r in self.reqs.values() if r.state != "done")
            left = max(0, min(left, c.kv_token_budget - held))
        for r in queue:
            if left <= 0:
                break
            n = min(r.prompt - r.prefill_done, left)
            slices.append((r.id, r.prefill_done, n))
            left -= n
            if not c.multi_fill:
                break
        pred = self.iter_time([(o, n) for _, o, n in slices], ctx)
        if c.dynamic_chunk and slices and pred > slack + 1e-12 * max(1.0, abs(slack)):
            rid, o, n = slices[-1]
            lo, hi = 0, n
            while hi - lo > 1:
                mid = (lo + hi) // 2
                t = self.iter_time([(a, b) for _, a, b in slices[:-1]] + [(o, mid)], ctx)
                if t <= slack + 1e-12 * max(1.0, abs(slack)):
                    lo = mid
                else:
                    hi = mid
            slices = slices[:-1] + ([(rid, o, lo)] if lo > 0 else [])
            pred = self.iter_time([(a, b) for _, a, b in slices], ctx)
        b = Batch(slices, dec, budget, pred, slack, infeasible, relegated)
        self.last = b
        return b

    def max_chunk(self, ctx: Sequence[int], offset: int, slack: float, cap: int) -> Tuple[int, bool]:
        """S:116-124 by bisection (oracle.predictor.max_feasible_chunk's rule)."""
        def ok(C):
            return self.iter_time([(offset, C)] if C else [], ctx) <= slack + 1e-12 * max(1.0, abs(slack))
        if not ok(0):
            return 0, True
        if ok(cap):
            return cap, False
        lo, hi = 0, cap
        while hi - lo > 1:
            mid = (lo + hi) // 2
            if ok(mid):
                lo = mid
            else:
                hi = mid
        return lo, False

    # ---- ⑦ completion ----
    def complete(self, now: float, finished: Sequence[int]) -> List[int]:
        """The last batch ran and ended at `now`; `finished` = its decodes that emitted their
        last token (the engine's EOS).  Returns the ids completed."""
        b = self.last
        if b is None:
            raise ValueError("no batch outstanding")
        fin = set(finished)
        if fin - {rid for rid, _ in b.decodes}:
            raise ValueError("finished id not among the batch's decodes")
        self.last = None
        done = []
        for rid, ctx in b.decodes:
            r = self.reqs[rid]
            r.decoded += 1
            r.tokens.append(now)
            if rid in fin:
                r.state = "done"
                self.hist.add(r.app, r.decoded)
                done.append(rid)
        last_prefill = None
        for rid, o, n in b.slices:
            r = self.reqs[rid]
            r.prefill_done += n
            last_prefill = rid
            if r.prefill_done == r.prompt:
                r.state = "decode"
        self.inflight = None
        if last_prefill is not None and self.reqs[last_prefill].state in ("prefill", "relegated"):
            self.inflight = last_prefill
        return done


class AffineModel:
    """SPEC's cost model: c0 + c1 * (prefill tokens + decodes) + c2 * sum ctx."""

    def __init__(self, c0: float, c1: float, c2: float):
        self.c0, self.c1, self.c2 = c0, c1, c2

    def iter_time(self, slices, decode_ctx) -> float:
        tok = sum(n for _, n in slices) + len(decode_ctx)
        return self.c0 + self.c1 * tok + self.c2 * float(sum(decode_ctx))


def simulate(sched: Scheduler, trace, qos_of, exec_time=None, max_iters: int = 10_000_000):
    """SPEC's single-replica event loop: admit arrivals up to `now`, build the batch,
    advance `now` by its execution time (default: the predicted latency), complete it.
    `trace` items carry id, t_arrival, prompt, decode (ground truth), bucket, low, app;
    `qos_of(bucket) -> QoS`.  Returns the iteration log [(now_start, batch, dt)]."""
    reqs = sorted(trace, key=lambda r: (r.t_arrival, r.id))
    truth = {r.id: r.decode for r in reqs}
    now, i, log = 0.0, 0, []
    for _ in range(max_iters):
        while i < len(reqs) and reqs[i].t_arrival <= now:
            r = reqs[i]
            sched.submit(Req(r.id, r.t_arrival, r.prompt, qos_of(r.bucket), r.low, r.app))
            i += 1
        b = sched.next_batch(now)
        if not b.slices and not b.decodes:
            sched.last = None
            if i >= len(reqs):
                break
            now = max(now, reqs[i].t_arrival)
            continue
        dt = b.predicted if exec_time is None else exec_time(b)
        log.append((now, b, dt))
        now += dt
        fin = [rid for rid, _ in b.decodes if sched.reqs[rid].decoded + 1 == truth[rid]]
        sched.complete(now, fin)
    return log


def violations(sched: Scheduler):
    """Per-request verdicts against Eq. 1-3 (R18 "<=" passes): an interactive request
    is violated if any token n lands after D_n, a non-interactive one if its last token
    lands after D_total; a relegated request counts as violated."""
    out = {}
    for r in sched.reqs.values():
        if r.relegated:
            out[r.id] = True
        elif r.qos.interactive:
            out[r.id] = any(t > deadline_token(r.t_arrival, r.qos.slo_ttft, r.qos.slo_tbt, n) + 1e-12 * max(1.0, t)
                            for n, t in enumerate(r.tokens, start=1))
        else:
            out[r.id] = bool(r.tokens) and r.tokens[-1] > deadline_total(r.t_arrival, r.qos.slo_ttlt) + 1e-12 * max(1.0, r.tokens[-1])
    return out

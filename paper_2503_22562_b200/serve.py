"""One serving replica: the QoS scheduler core
(`niyama_sched_*`, C++) picks each iteration's hybrid batch, the engine runs it
through every layer on the GPU (`niyama_kv_append` + `niyama_hybrid_attention`
per layer, the real kernels), and the replica's clock advances by the MEASURED
device time of the iteration (PAPER.md P:205 steps ①-⑦).

The engine is attention-only (no linear layers: §8(f) rank 4); activations are
synthetic (seeded random Q/K/V rows, the same buffers every iteration).  The
decode lengths of a trace are ground truth known only to the engine (the
engine's EOS, "decode length is unknown").  A `ModelExecutor` replaces the
GPU by the predictor's own estimate (the SPEC simulator) for capacity
searches.  Metrics follow SPEC's report: TTFT = first token -
arrival, violations against Eq. 1-3 with "<=" passing (R18), relegated requests
count as violated.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from ._binding import KVCache, NiyamaError, Predictor, Scheduler, ENOBLOCKS


@dataclass
class QoSBucket:
    interactive: bool
    slo_ttft: float = 0.0
    slo_tbt: float = 0.0
    slo_ttlt: float = 0.0


@dataclass
class IterRecord:
    t_start: float
    seconds: float            # measured (GPU) or predicted (model executor)
    predicted: float          # the scheduler's prediction for the batch
    prefill_tokens: int
    decodes: int
    slices: int
    budget: int
    infeasible: bool
    relegated: int
    attention_s: float = float("nan")   # GPU: the attention launches alone (what the predictor models)


@dataclass
class ReqRecord:
    id: int
    t_arrival: float
    prompt: int
    decode: int
    bucket: int
    low: bool
    tokens: List[float] = field(default_factory=list)
    relegated: bool = False


class ModelExecutor:
    """The predictor's estimate as the execution time (no GPU)."""

    def __init__(self, predictor: Predictor, layers: float = 1.0, fixed_s: float = 0.0):
        self.pred, self.layers, self.fixed_s = predictor, layers, fixed_s

    def run(self, batch) -> float:
        return self.fixed_s + self.layers * self.pred.predict(batch.desc())

    def release(self, seq: int):
        pass


class GpuExecutor:
    """n_layers x (append + attention) of the batch on cuda:device, timed with CUDA events."""

    def __init__(self, shape, n_layers: int, num_blocks: int, max_rows: int = 2048 + 512, device: int = 0,
                 seed: int = 0, linear=None, head_start_us: float = 0.0):
        """linear: optional callable object with pre(h) -> (q, k, v) and post(h, o, T) -> h (a model's
        linear layers, e.g. cuBLAS GEMMs) run around every layer's append + attention.
        head_start_us > 0: the stream spins that long (torch.cuda._sleep, before the timed region)
        so the host enqueues the whole iteration before the GPU starts it; otherwise a batch whose
        kernels are shorter than the binding's per-launch host cost is timed with the host's
        launch gaps inside (tools/replay_outliers.py)."""
        import torch
        self.torch = torch
        self.n_layers = n_layers
        self.kv = KVCache(n_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, num_blocks,
                          block_size=shape.block_size, dtype="bf16", device=device)
        g = torch.Generator(device=f"cuda:{device}")
        g.manual_seed(seed)
        dev = f"cuda:{device}"
        self.max_rows = max_rows
        mk = lambda *s: torch.randn(*s, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)  # noqa: E731
        self.q = mk(max_rows, shape.num_q_heads, shape.head_dim)
        self.k = mk(max_rows, shape.num_kv_heads, shape.head_dim)
        self.v = mk(max_rows, shape.num_kv_heads, shape.head_dim)
        self.obuf = torch.empty(shape.num_q_heads * max_rows * shape.head_dim, dtype=torch.bfloat16, device=dev)
        self.hq, self.d = shape.num_q_heads, shape.head_dim
        self.stream = torch.cuda.current_stream(device)
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)
        self.ev_attn = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                        for _ in range(n_layers)]
        self.last_attention_s = 0.0
        self.launches = 0
        self.linear = linear
        self.head_start_cycles = int(head_start_us * 2000.0)   # ~2 GHz SM clock

    def run(self, batch) -> float:
        T = sum(n for _, _, n in batch.slices) + len(batch.decodes)
        if T > self.max_rows:
            raise ValueError(f"batch of {T} rows exceeds the engine's buffers ({self.max_rows})")
        plan = self.kv.plan(batch.desc(), self.stream)
        q, k, v = self.q[:T], self.k[:T], self.v[:T]
        o = self.obuf[:self.hq * T * self.d].view(self.hq, T, self.d)
        h = self.linear.x[:T] if self.linear is not None else None
        if self.head_start_cycles > 0:
            with self.torch.cuda.stream(self.stream):
                self.torch.cuda._sleep(self.head_start_cycles)
        self.e0.record(self.stream)
        for layer in range(self.n_layers):
            if self.linear is not None:
                q, k, v = self.linear.pre(h)
            self.kv.append(plan, layer, k, v, self.stream)
            a, b = self.ev_attn[layer]
            a.record(self.stream)
            self.kv.attention(plan, layer, q, o, None, 0.0, self.stream)
            b.record(self.stream)
            if self.linear is not None:
                h = self.linear.post(h, o, T)
        self.e1.record(self.stream)
        plan.close()
        self.e1.synchronize()
        self.launches += 2 * self.n_layers
        self.last_attention_s = sum(a.elapsed_time(b) for a, b in self.ev_attn) * 1e-3
        return self.e0.elapsed_time(self.e1) * 1e-3

    def release(self, seq: int):
        self.kv.release(seq)


def replay(sched: Scheduler, executor, trace: Sequence, buckets: Sequence[QoSBucket], until: float = math.inf,
           max_iters: int = 10_000_000, record: Optional[list] = None):
    """The serving loop (SPEC's event loop): admit arrivals up to `now`, build the
    batch, execute it, advance `now`, complete it.  Returns (iterations, requests)."""
    reqs = sorted(trace, key=lambda r: (r.t_arrival, r.id))
    recs: Dict[int, ReqRecord] = {}
    iters: List[IterRecord] = []
    now, i = 0.0, 0
    decoded: Dict[int, int] = {}
    for _ in range(max_iters):
        while i < len(reqs) and reqs[i].t_arrival <= now:
            r = reqs[i]
            b = buckets[r.bucket]
            sched.submit(r.id, r.t_arrival, r.prompt, b.interactive, b.slo_ttft, b.slo_tbt, b.slo_ttlt, r.low,
                         r.app, r.bucket)
            recs[r.id] = ReqRecord(r.id, r.t_arrival, r.prompt, r.decode, r.bucket, r.low)
            decoded[r.id] = 0
            i += 1
        if now > until:
            break
        batch = sched.next_batch(now)
        for rid in batch.relegated:
            recs[rid].relegated = True
        if batch.empty:
            if i >= len(reqs):
                break
            now = max(now, reqs[i].t_arrival)
            continue
        if record is not None:  # the batch descriptors (predictor calibration on the engine's own iterations)
            record.append(batch.desc())
        dt = executor.run(batch)
        iters.append(IterRecord(now, dt, batch.predicted, sum(n for _, _, n in batch.slices), len(batch.decodes),
                                len(batch.slices), batch.budget, batch.infeasible, len(batch.relegated),
                                getattr(executor, "last_attention_s", float("nan"))))
        now += dt
        fin = []
        for rid, _ in batch.decodes:
            decoded[rid] += 1
            recs[rid].tokens.append(now)
            if decoded[rid] == recs[rid].decode:
                fin.append(rid)
        sched.complete(now, fin)
        for rid in fin:
            executor.release(rid)
    return iters, recs


def verdicts(recs: Dict[int, ReqRecord], buckets: Sequence[QoSBucket], t_end: float = math.inf):
    """Per request: violated? (Eq. 1-3, R18 "<=" passes; relegated counts as violated; an unfinished
    request is violated if the deadline of its next token (interactive) or its completion deadline
    (non-interactive) has passed by t_end)."""
    out = {}
    for r in recs.values():
        b = buckets[r.bucket]
        tbt_miss = 0
        done = len(r.tokens) == r.decode
        if b.interactive:
            bad = False
            for n, t in enumerate(r.tokens, start=1):
                d = r.t_arrival + b.slo_ttft + (n - 1) * b.slo_tbt
                if t > d + 1e-12 * max(1.0, t):
                    bad = True
                    tbt_miss += n > 1
            if not done and r.t_arrival + b.slo_ttft + len(r.tokens) * b.slo_tbt < t_end:
                bad = True
        else:
            bad = bool(r.tokens) and r.tokens[-1] > r.t_arrival + b.slo_ttlt + 1e-12 * max(1.0, r.tokens[-1])
            if not done and r.t_arrival + b.slo_ttlt < t_end:
                bad = True
        out[r.id] = dict(violated=bad or r.relegated, relegated=r.relegated, finished=len(r.tokens) == r.decode,
                         tbt_miss=tbt_miss)
    return out


def summarize(iters: List[IterRecord], recs: Dict[int, ReqRecord], buckets: Sequence[QoSBucket],
              t_end: Optional[float] = None, fixed_s: float = 0.0) -> dict:
    span = (t_end if t_end is not None else (iters[-1].t_start + iters[-1].seconds if iters else 0.0))
    v = verdicts(recs, buckets, span)
    done = [r for r in recs.values() if v[r.id]["finished"]]
    judged = [r for r in recs.values() if v[r.id]["finished"] or v[r.id]["violated"]]
    def pct(xs):
        return 100.0 * float(np.mean(xs)) if len(xs) else 0.0
    by_bucket = {str(k): pct([v[r.id]["violated"] for r in judged if r.bucket == k]) for k in range(len(buckets))}
    hi = [v[r.id]["violated"] for r in judged if not r.low]
    lo = [v[r.id]["violated"] for r in judged if r.low]
    err = np.array([it.predicted / it.seconds - 1.0 for it in iters]) if iters else np.zeros(0)
    # attention alone: the scheduler's prediction minus its fixed per-iteration part
    att = np.array([(it.predicted - fixed_s) / it.attention_s - 1.0 for it in iters
                    if it.attention_s == it.attention_s and it.attention_s > 0])
    chunks = np.array([it.prefill_tokens for it in iters])
    edges = [0, 1, 257, 513, 1025, 1537, 2049]
    hist = {f"{a}-{b - 1}": int(np.sum((chunks >= a) & (chunks < b))) for a, b in zip(edges[:-1], edges[1:])}
    tokens = sum(len(r.tokens) for r in recs.values() if buckets[r.bucket].interactive)
    ttft = [r.tokens[0] - r.t_arrival for r in recs.values() if r.tokens]
    good = sum(1 for r in done if not v[r.id]["violated"])
    return {
        "requests": len(recs), "finished": len(done), "judged": len(judged),
        "violations_pct": pct([v[r.id]["violated"] for r in judged]),
        "violations_pct_by_bucket": by_bucket,
        "violations_pct_high_priority": pct(hi), "violations_pct_low_priority": pct(lo),
        "relegated_pct": pct([v[r.id]["relegated"] for r in recs.values()]),
        "tbt_miss_pct_of_interactive_tokens": 100.0 * sum(v[r.id]["tbt_miss"] for r in recs.values()) / max(1, tokens),
        "ttft_p50_s": float(np.median(ttft)) if ttft else None,
        "ttft_p99_s": float(np.percentile(ttft, 99)) if ttft else None,
        "goodput_rps": good / span if span > 0 else 0.0,
        "iterations": len(iters), "simulated_s": span,
        "predictor_rel_err": ({"p50": float(np.median(np.abs(err))), "p95": float(np.percentile(np.abs(err), 95)),
                               "max": float(np.abs(err).max()), "mean_signed": float(err.mean())}
                              if len(err) else None),
        "predictor_rel_err_attention_only": ({"p50": float(np.median(np.abs(att))),
                                              "p95": float(np.percentile(np.abs(att), 95)),
                                              "max": float(np.abs(att).max()), "mean_signed": float(att.mean())}
                                             if len(att) else None),
        "chunk_histogram": hist,
        "mean_chunk": float(chunks.mean()) if len(chunks) else 0.0,
    }


__all__ = ["QoSBucket", "ModelExecutor", "GpuExecutor", "replay", "summarize", "verdicts", "IterRecord",
           "ReqRecord", "NiyamaError", "ENOBLOCKS"]

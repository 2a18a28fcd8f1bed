"""Seeded synthetic workloads for the hybrid-batch paged-attention path.

INPUT GENERATORS ONLY.  This module holds no attention, softmax, KV-cache or
block-table arithmetic: it draws request shapes and Q/K/V values from seeded
PCG64 streams and packages them as batch descriptors.  Both sides consume it —
the fp64 oracle (`oracle/`, test infrastructure) and the CUDA path
(`paper_2503_22562_b200`, through its C-ABI) — and neither imports the other.

Shapes follow SURVEY.md §8(d) "Config N inputs"; the batch structure follows
the paper's hybrid batch (§3.1 step ⑤: "a mixed batch of prefill
and decode tokens is constructed using the chosen prefill chunk and the
requests in the decode queue").  Length distributions follow the ShareGPT row
of Table 1 through the two-percentile lognormal fit of SPEC.md S:47
(sigma computed from the formula, reading R19).

Value recipe: Q, K, V ~ N(0, 1) drawn as float32 from PCG64(seed); for bf16
workloads they are rounded to bf16 with round-to-nearest-even and carried as
raw uint16 bit patterns (so that both sides see the identical stored bits).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

# ---------------------------------------------------------------------------
# data containers (no arithmetic)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Shape:
    """Per-layer attention shape.  dtype is the stored KV/Q/O type."""

    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    block_size: int = 16
    dtype: str = "bf16"  # "bf16" | "f32"
    num_layers: int = 1

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def elt_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    @property
    def np_store(self):
        return np.uint16 if self.dtype == "bf16" else np.float32


@dataclass
class BatchDesc:
    """One iteration's hybrid batch (mirrors `niyama_batch_desc`, include/niyama.h).

    Rows are ordered prefill slices first (slice i contributes prefill_len[i]
    rows at positions prefill_offset[i] .. +len-1), then one row per decode
    whose new token sits at position decode_ctx[j]-1 (R4, R6).
    """

    prefill_seq: List[int] = field(default_factory=list)
    prefill_offset: List[int] = field(default_factory=list)
    prefill_len: List[int] = field(default_factory=list)
    decode_seq: List[int] = field(default_factory=list)
    decode_ctx: List[int] = field(default_factory=list)
    tier: Optional[List[int]] = None

    @property
    def num_prefill(self) -> int:
        return len(self.prefill_seq)

    @property
    def num_decode(self) -> int:
        return len(self.decode_seq)

    @property
    def num_rows(self) -> int:
        return int(sum(self.prefill_len)) + len(self.decode_seq)

    def tiers(self) -> List[int]:
        if self.tier is None:
            return [0] * (self.num_prefill + self.num_decode)
        return list(self.tier)


@dataclass
class Step:
    """A batch plus its new-token tensors in stored representation.

    q: [T][Hq][d] or None (fill-only step: KV append without attention)
    k, v: [T][Hkv][d]
    """

    desc: BatchDesc
    k: np.ndarray
    v: np.ndarray
    q: Optional[np.ndarray] = None


@dataclass
class Workload:
    name: str
    shape: Shape
    steps: List[Step]
    num_blocks: int

    @property
    def final(self) -> Step:
        return self.steps[-1]


# ---------------------------------------------------------------------------
# value generation
# ---------------------------------------------------------------------------


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (round-to-nearest-even) and return the uint16 bits.
    Input representation only (finite normal draws)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    bias = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + bias) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def draw_values(g: np.random.Generator, shape, dtype: str, scale: float = 1.0) -> np.ndarray:
    x = g.standard_normal(size=shape, dtype=np.float32)
    if scale != 1.0:
        x *= np.float32(scale)
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    return x


def make_step(g: np.random.Generator, shape: Shape, desc: BatchDesc, with_q: bool = True,
              q_scale: float = 1.0) -> Step:
    T = desc.num_rows
    k = draw_values(g, (T, shape.num_kv_heads, shape.head_dim), shape.dtype)
    v = draw_values(g, (T, shape.num_kv_heads, shape.head_dim), shape.dtype)
    q = draw_values(g, (T, shape.num_q_heads, shape.head_dim), shape.dtype, q_scale) if with_q else None
    return Step(desc=desc, k=k, v=v, q=q)


def blocks_needed(lengths, block_size: int) -> int:
    """Capacity sizing for the pool (ceil per sequence) — used to size num_blocks."""
    return int(sum((int(n) + block_size - 1) // block_size for n in lengths))


def fill_step(g, shape: Shape, seqs, lengths) -> Step:
    """Fill-only step: one prefill slice per sequence from offset 0."""
    desc = BatchDesc(prefill_seq=list(seqs), prefill_offset=[0] * len(seqs),
                     prefill_len=[int(n) for n in lengths])
    return make_step(g, shape, desc, with_q=False)


# ---------------------------------------------------------------------------
# SURVEY §8(d) configs
# ---------------------------------------------------------------------------

TINY = Shape(num_q_heads=4, num_kv_heads=2, head_dim=64, block_size=16, dtype="f32")
L8B = Shape(num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
L70B = Shape(num_q_heads=64, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")


def hybrid(shape: Shape, name: str, *, prefill_offset: int, chunk: int, decode_ctx, seed: int,
           q_scale: float = 1.0, prefill_seq: int = 0, extra_blocks: int = 0,
           tiers=None) -> Workload:
    """Generic 'prefix fill, then one hybrid batch' workload.

    Sequence `prefill_seq` is pre-filled to `prefill_offset` tokens, then
    decode sequences 1..D are pre-filled to ctx-1; the final step is the hybrid
    batch: one chunk of `chunk` rows at `prefill_offset` plus one decode row per
    sequence at its ctx (P:205 ⑤)."""
    decode_ctx = [int(c) for c in decode_ctx]
    D = len(decode_ctx)
    dseqs = [prefill_seq + 1 + j for j in range(D)]
    g = rng(seed)
    steps = []
    fill_seqs = ([prefill_seq] if chunk > 0 or prefill_offset > 0 else []) + dseqs
    fill_lens = ([prefill_offset] if chunk > 0 or prefill_offset > 0 else []) + [c - 1 for c in decode_ctx]
    if fill_seqs:
        steps.append(fill_step(g, shape, fill_seqs, fill_lens))
    desc = BatchDesc(
        prefill_seq=[prefill_seq] if chunk > 0 else [],
        prefill_offset=[prefill_offset] if chunk > 0 else [],
        prefill_len=[chunk] if chunk > 0 else [],
        decode_seq=dseqs, decode_ctx=decode_ctx,
        tier=tiers)
    steps.append(make_step(g, shape, desc, with_q=True, q_scale=q_scale))
    final_lens = ([prefill_offset + chunk] if chunk > 0 else []) + decode_ctx
    nb = blocks_needed(final_lens, shape.block_size) + extra_blocks
    return Workload(name=name, shape=shape, steps=steps, num_blocks=max(nb, 1))


def config1_tiny(variant: str = "aligned", peaky: bool = False, seed: int = 1) -> Workload:
    """Config 1: Hq=4, Hkv=2, d=64, B=16, fp32; one 64-token chunk
    (variant 'unaligned': o=37, c=27) plus decodes at ctx 17/100/255."""
    o, c = (0, 64) if variant == "aligned" else (37, 27)
    return hybrid(TINY, f"tiny-{variant}{'-peaky' if peaky else ''}", prefill_offset=o, chunk=c,
                  decode_ctx=[17, 100, 255], seed=seed, q_scale=8.0 if peaky else 1.0)


def l8b_decode_ctx(num_decode: int = 64, max_ctx: int = 4096, seed: int = 0) -> np.ndarray:
    """Decode contexts ~ U{1..max_ctx} from PCG64(seed) (ΣL = 133,674 at seed 0)."""
    return rng(seed).integers(1, max_ctx + 1, size=num_decode)


def config2_l8b(prefill_offset: int = 1536, chunk: int = 512, ctx_mode: str = "uniform",
                num_decode: int = 64, seed: int = 2, shape: Shape = L8B) -> Workload:
    """Config 2: Llama-3-8B attention shapes, bf16; chunk 512 at o=1536 + 64 decodes,
    ctx ~ U{1..4096} (seed 0) or all 4096."""
    if ctx_mode == "uniform":
        ctx = l8b_decode_ctx(num_decode)
    else:
        ctx = np.full(num_decode, 4096)
    return hybrid(shape, f"l8b-c{chunk}-o{prefill_offset}-{ctx_mode}", prefill_offset=prefill_offset,
                  chunk=chunk, decode_ctx=ctx, seed=seed)


def config4_l70b(prefill_offset: int = 6144, chunk: int = 2048, num_decode: int = 128,
                 ctx: int = 8192, seed: int = 4) -> Workload:
    """Config 4: Llama-3-70B attention shapes (64 q / 8 kv heads), 2048 chunk + 128 decodes at 8K."""
    return hybrid(L70B, f"l70b-c{chunk}-o{prefill_offset}", prefill_offset=prefill_offset, chunk=chunk,
                  decode_ctx=[ctx] * num_decode, seed=seed)


# ShareGPT (Table 1): prompt p50/p90 = 1730/5696, decode p50/p90 = 415/834.
SHAREGPT = dict(prompt=(1730, 5696), decode=(415, 834))
Z90 = 1.2815515655446004  # standard-normal 0.9 quantile


def lognormal_fit(p50: float, p90: float):
    """SPEC S:47 fit_lognormal: mu = ln p50, sigma = (ln p90 - ln p50) / z_0.9."""
    mu = math.log(p50)
    sigma = 0.0 if p50 == p90 else (math.log(p90) - math.log(p50)) / Z90
    return mu, sigma


def sweep_point(chunk: int, num_decode: int, seed: int, shape: Shape = L8B, max_ctx: int = 8192) -> Workload:
    """Config 3 point: offset drawn from the ShareGPT prompt lognormal as a chunk-aligned
    offset below the prompt; decode ctx = prompt + U[0, decode) clipped to [1, max_ctx]."""
    g = rng(1000 + seed)
    mu_p, sd_p = lognormal_fit(*SHAREGPT["prompt"])
    mu_d, sd_d = lognormal_fit(*SHAREGPT["decode"])
    prompt = int(min(max(round(g.lognormal(mu_p, sd_p)), chunk + 1), max_ctx))
    n_chunks = max(0, (prompt - 1) // chunk)
    o = int(g.integers(0, n_chunks + 1)) * chunk if n_chunks > 0 else 0
    o = min(o, max_ctx - chunk)
    prompts = np.clip(np.round(g.lognormal(mu_p, sd_p, size=num_decode)), 1, max_ctx)
    decs = np.round(g.lognormal(mu_d, sd_d, size=num_decode))
    ctx = np.clip(prompts + np.floor(g.random(num_decode) * np.maximum(decs, 1)), 1, max_ctx).astype(int)
    return hybrid(shape, f"sweep-c{chunk}-D{num_decode}-s{seed}", prefill_offset=o, chunk=chunk,
                  decode_ctx=ctx, seed=seed + 77)


def revalue(wl: Workload, seed: int, q_scale: float = 1.0) -> Workload:
    """The same batches (descriptors, shapes) with fresh Q/K/V values from PCG64(seed):
    another layer of the same iterations (a model's layers see the same batch
    composition with different activations)."""
    g = rng(seed)
    steps = [make_step(g, wl.shape, st.desc, with_q=st.q is not None, q_scale=q_scale) for st in wl.steps]
    return Workload(name=f"{wl.name}-v{seed}", shape=wl.shape, steps=steps, num_blocks=wl.num_blocks)


def random_hybrid(shape: Shape, seed: int, *, num_prefill: int = 1, max_chunk: int = 300,
                  num_decode: int = 8, max_ctx: int = 700, q_scale: float = 1.0,
                  extra_blocks: int = 0) -> Workload:
    """Small ragged hybrid batch for parity tests: several prefill slices at random
    (unaligned) offsets and decodes at random contexts (multi-slice reading R2)."""
    g = rng(seed)
    offs = [int(x) for x in g.integers(0, max_ctx, size=num_prefill)]
    lens = [int(x) for x in g.integers(1, max_chunk + 1, size=num_prefill)]
    ctx = [int(x) for x in g.integers(1, max_ctx + 1, size=num_decode)]
    pseqs = list(range(num_prefill))
    dseqs = list(range(num_prefill, num_prefill + num_decode))
    steps = []
    fill_seqs = pseqs + dseqs
    fill_lens = offs + [c - 1 for c in ctx]
    steps.append(fill_step(g, shape, fill_seqs, fill_lens))
    tiers = [int(x) for x in g.integers(0, 3, size=num_prefill + num_decode)]
    desc = BatchDesc(prefill_seq=pseqs, prefill_offset=offs, prefill_len=lens,
                     decode_seq=dseqs, decode_ctx=ctx, tier=tiers)
    steps.append(make_step(g, shape, desc, with_q=True, q_scale=q_scale))
    nb = blocks_needed([o + c for o, c in zip(offs, lens)] + ctx, shape.block_size) + extra_blocks
    return Workload(name=f"random-s{seed}", shape=shape, steps=steps, num_blocks=nb)


# ---------------------------------------------------------------------------
# config 5: QoS-tiered arrival traces (inputs of the scheduler; no method arithmetic)
# ---------------------------------------------------------------------------

# Table 3: three equal buckets; Q1 interactive TTFT 6 s / TBT 50 ms,
# Q2 / Q3 non-interactive TTLT 600 s / 1800 s.
TABLE3 = [dict(interactive=True, slo_ttft=6.0, slo_tbt=0.050, slo_ttlt=0.0, share=1 / 3),
          dict(interactive=False, slo_ttft=0.0, slo_tbt=0.0, slo_ttlt=600.0, share=1 / 3),
          dict(interactive=False, slo_ttft=0.0, slo_tbt=0.0, slo_ttlt=1800.0, share=1 / 3)]


@dataclass
class TraceRequest:
    id: int
    t_arrival: float
    prompt: int
    decode: int          # ground truth (the engine's EOS), hidden from the scheduler
    bucket: int          # index into the trace's bucket list
    low: bool            # application hint "low priority" (20% per bucket)
    app: int             # decode-length history key = bucket (one application per bucket)


def qos_trace(duration_s: float, qps_schedule, seed: int, dataset=SHAREGPT, low_fraction: float = 0.2,
              buckets=TABLE3, max_prompt: Optional[int] = None, max_decode: Optional[int] = None) -> List[TraceRequest]:
    """Poisson arrivals with a piecewise-constant rate: qps_schedule = [(t_start,
    qps), ...] (inclusive start; P:534's diurnal low/high steps), or a single qps.  Token
    counts from the dataset's two-percentile lognormals (Table 1), rounded, >= 1
    (optionally capped); bucket by the shares; Low priority with probability
    low_fraction within each bucket.  Deterministic given seed (PCG64)."""
    if not isinstance(qps_schedule, (list, tuple)):
        qps_schedule = [(0.0, float(qps_schedule))]
    g = rng(seed)
    mu_p, sd_p = lognormal_fit(*dataset["prompt"])
    mu_d, sd_d = lognormal_fit(*dataset["decode"])
    shares = np.cumsum([b["share"] for b in buckets])
    out: List[TraceRequest] = []
    steps = list(qps_schedule) + [(duration_s, 0.0)]
    for (t0, qps), (t1, _) in zip(steps[:-1], steps[1:]):
        t = t0
        while qps > 0:
            t += g.exponential(1.0 / qps)
            if t >= min(t1, duration_s):
                break
            p = max(1, int(round(g.lognormal(mu_p, sd_p))))
            d = max(1, int(round(g.lognormal(mu_d, sd_d))))
            if max_prompt:
                p = min(p, max_prompt)
            if max_decode:
                d = min(d, max_decode)
            b = int(np.searchsorted(shares, g.random() * shares[-1], side="right"))
            low = bool(g.random() < low_fraction)
            out.append(TraceRequest(len(out), float(t), p, d, min(b, len(buckets) - 1), low, min(b, len(buckets) - 1)))
    return out


def diurnal_schedule(duration_s: float, low_qps: float, high_qps: float, period_s: float = 900.0):
    """load alternates between low and high every 15 minutes."""
    sched, t, hi = [], 0.0, False
    while t < duration_s:
        sched.append((t, high_qps if hi else low_qps))
        t += period_s
        hi = not hi
    return sched

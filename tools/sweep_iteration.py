"""§8(f) rank 4 — full-iteration measurements (Fig. 4 analogue and the full-iteration predictor).

A Llama-3-8B iteration on one B200: 32 layers x [RMSNorm -> QKV GEMM -> KV append ->
hybrid attention (this library) -> O GEMM -> residual -> RMSNorm -> gate/up GEMM -> SiLU*mul
-> down GEMM -> residual], weights random bf16 (synthetic; the GEMMs are cuBLAS through
torch.matmul: plain library GEMMs), one weight set reused by every layer (436 MB per
layer, far above the 126 MB L2, so it is streamed every layer as in a real model).

Measures, with CUDA events on the device:
  * the linear part alone per token count T (the GEMM + elementwise work of one layer);
  * full iterations on config-3-like batches (chunk c at offset o + D decodes, ShareGPT-like
    contexts), split into train (seeds 0, 1 + random) and held-out (seed 2 + off-grid).
Writes the raw JSON; tools/fit_iteration.py fits and compares predictors (CPU).

    python tools/sweep_iteration.py [--layers 32] [--out gpurun_out/iteration_sweep.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
import workloads as W  # noqa: E402
from sweep_predictor import point_desc  # noqa: E402

HID, INTER, HQ, HKV, D = 4096, 14336, 32, 8, 128


class LinearLayers:
    """One Llama-3-8B layer's linear part (weights shared by every layer); the serve.GpuExecutor
    `linear` protocol: x (activations buffer), pre(h) -> (q, k, v), post(h, o, T) -> h."""

    def __init__(self, max_t=4096 + 256):
        g = torch.Generator(device="cuda")
        g.manual_seed(0)
        mk = lambda *s, sc=0.02: (torch.randn(*s, generator=g, device="cuda") * sc).to(torch.bfloat16)  # noqa: E731
        self.w_qkv = mk(HID, (HQ + 2 * HKV) * D)
        self.w_o = mk(HQ * D, HID)
        self.w_gu = mk(HID, 2 * INTER)
        self.w_d = mk(INTER, HID)
        self.ln = torch.ones(HID, device="cuda", dtype=torch.bfloat16)
        self.x = mk(max_t, HID, sc=1.0)

    @staticmethod
    def rms(x, w):
        v = x.float().pow(2).mean(-1, keepdim=True)
        return (x.float() * torch.rsqrt(v + 1e-5)).to(torch.bfloat16) * w

    def pre(self, h):
        qkv = self.rms(h, self.ln) @ self.w_qkv
        q = qkv[:, :HQ * D].reshape(-1, HQ, D)
        k = qkv[:, HQ * D:(HQ + HKV) * D].reshape(-1, HKV, D)
        v = qkv[:, (HQ + HKV) * D:].reshape(-1, HKV, D)
        return q.contiguous(), k.contiguous(), v.contiguous()

    def post(self, h, o, T):
        a = o.reshape(HQ, T, D).permute(1, 0, 2).reshape(T, HQ * D)   # head-major O -> token-major
        h = h + a @ self.w_o
        gu = self.rms(h, self.ln) @ self.w_gu
        act = torch.nn.functional.silu(gu[:, :INTER]) * gu[:, INTER:]
        return h + act @ self.w_d


class Model:
    def __init__(self, layers, num_blocks, max_t=4096 + 256):
        self.lin = LinearLayers(max_t)
        self.layers = layers
        self.kv = ny.KVCache(layers, HQ, HKV, D, num_blocks, block_size=16, dtype="bf16", device=0)
        self.x = self.lin.x
        self.obuf = torch.zeros(HQ * max_t * D, device="cuda", dtype=torch.bfloat16)

    def linear_pre(self, h):
        return self.lin.pre(h)

    def linear_post(self, h, o, T):
        return self.lin.post(h, o, T)

    def iteration(self, plan, T, attention=True):
        h = self.x[:T]
        o = self.obuf[:HQ * T * D].view(HQ, T, D)
        for layer in range(self.layers):
            q, k, v = self.linear_pre(h)
            if attention:
                self.kv.append(plan, layer, k, v)
                self.kv.attention(plan, layer, q, o)
            h = self.linear_post(h, o, T)
        return h


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts), ts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--random", type=int, default=40)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "iteration_sweep.json"))
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
    max_dec = 128
    free, _ = torch.cuda.mem_get_info()
    blocks = int((free - (12 << 30)) // (args.layers * 65536))   # leave room for weights and activations
    blocks = min(blocks, max_dec * 8192 // 16 + 4096)
    print(f"KV pool: {blocks} blocks x {args.layers} layers", flush=True)
    m = Model(args.layers, num_blocks=blocks)
    t0 = time.time()
    # linear part alone, per token count
    lin = []
    for T in (16, 32, 64, 128, 192, 256, 384, 512, 768, 1024, 1536, 2048, 2304, 3072, 4096):
        plan_dummy = None
        med, _ = timed(lambda: m.iteration(plan_dummy, T, attention=False), args.reps)
        lin.append(dict(T=T, seconds=med))
        print(f"linear T={T:5d} {med * 1e3:8.3f} ms / iteration", flush=True)
    rows = []

    def run(kind, seed, chunk, nd):
        o, ctx = point_desc(max(chunk, 1), nd, seed)
        if chunk == 0:
            o = 0
        seqs = list(range(1, len(ctx) + 1))
        fill = W.BatchDesc(prefill_seq=[0] + seqs, prefill_offset=[0] * (1 + len(ctx)),
                           prefill_len=[o] + [c - 1 for c in ctx])
        kv = m.kv
        p = kv.plan(fill)
        Tf = fill.num_rows
        k = torch.randn(min(Tf, 65536), HKV, D, device="cuda").to(torch.bfloat16)
        kbuf = k.repeat((Tf + k.shape[0] - 1) // k.shape[0], 1, 1)[:Tf].contiguous()
        for layer in range(args.layers):
            kv.append(p, layer, kbuf, kbuf)
        desc = W.BatchDesc(prefill_seq=[0] if chunk else [], prefill_offset=[o] if chunk else [],
                           prefill_len=[chunk] if chunk else [], decode_seq=seqs, decode_ctx=ctx)
        plan = kv.plan(desc)
        T = desc.num_rows
        m.iteration(plan, T)
        med, ts = timed(lambda: m.iteration(plan, T), args.reps)
        plan.rollback()   # replay: the timed iterations re-append at the same positions
        plan.close()
        p.close()
        for sq in [0] + seqs:
            kv.release(sq)
        rows.append(dict(kind=kind, seed=seed, chunk=chunk, offset=o, D=nd, ctx=ctx, sum_ctx=int(sum(ctx)), T=T,
                         seconds=med, spread=(max(ts) - min(ts)) / med))
        print(f"{kind:7s} s={seed:4d} c={chunk:5d} o={o:5d} D={nd:3d} T={T:5d} iter={med * 1e3:8.3f} ms "
              f"tok/s={T / med:10.0f}", flush=True)

    for seed in range(3):
        for chunk in (256, 512, 1024, 2048):
            for D in (16, 32, 64, 128):
                run("grid", seed, chunk, D)
    g = np.random.default_rng(7)
    for i in range(20):
        run("offgrid", 100 + i, int(g.integers(1, 2049)), int(g.integers(1, max_dec + 1)))
    g = np.random.default_rng(8)
    for i in range(args.random):
        run("random", 1000 + i, int(g.integers(0, 2049)), int(g.integers(1, max_dec + 1)))
    out = {"layers": args.layers, "model": "Llama-3-8B shapes (hidden 4096, 32 q / 8 kv heads, MLP 14336), bf16",
           "reps": args.reps, "timing": "median of reps, CUDA events around one full iteration (no L2 flush: the "
           "436 MB of weights per layer stream through L2 every layer)", "linear": lin, "points": rows,
           "wall_s": time.time() - t0, "device": torch.cuda.get_device_name(0)}
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Config 3 — dynamic-chunking sweep (a8 training and held-out data): measure the hybrid
attention launch on B200 over chunk {256, 512, 1024, 2048} x decodes {16, 32, 64, 128,
256} x 3 seeds (ShareGPT-like lengths, workloads.sweep_point), 40 off-grid points and
--train-random random points over the whole (c, D) space (incl. prefill-only and
decode-only batches).  Timing: CUDA events around ONE launch, median (and p10/p90) of
--reps reps, L2 flushed before every rep by reading a 512 MB buffer.  K/V values are
drawn on the device (timing only; parity is covered by tests/).  Writes the raw points;
tools/fit_predictor.py fits and evaluates (CPU, no GPU needed).

    python tools/sweep_predictor.py [--reps 50] [--raw profiles/r02/predictor_sweep_l8b.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2503_22562_b200 as ny  # noqa: E402


def point_desc(chunk, D, seed, max_ctx=8192):
    """Shapes of workloads.sweep_point without drawing K/V on the host."""
    g = W.rng(1000 + seed)
    mu_p, sd_p = W.lognormal_fit(*W.SHAREGPT["prompt"])
    mu_d, sd_d = W.lognormal_fit(*W.SHAREGPT["decode"])
    prompt = int(min(max(round(g.lognormal(mu_p, sd_p)), chunk + 1), max_ctx))
    n_chunks = max(0, (prompt - 1) // chunk)
    o = int(g.integers(0, n_chunks + 1)) * chunk if n_chunks > 0 else 0
    o = min(o, max_ctx - chunk)
    prompts = np.clip(np.round(g.lognormal(mu_p, sd_p, size=D)), 1, max_ctx)
    decs = np.round(g.lognormal(mu_d, sd_d, size=D))
    ctx = np.clip(prompts + np.floor(g.random(D) * np.maximum(decs, 1)), 1, max_ctx).astype(int).tolist()
    return o, ctx


class Rig:
    def __init__(self, shape, num_blocks, flush="read"):
        self.s = shape
        self.kv = ny.KVCache(1, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, num_blocks,
                             block_size=shape.block_size, dtype="bf16", device=0)
        # L2 flush by READING 512 MB (a write flush leaves ~126 MB of dirty lines whose
        # write-back lands inside the next timed launch: +~20 us and noise)
        self.scratch = torch.ones(256 << 20, dtype=torch.float16, device="cuda")
        self.sink = torch.empty((), dtype=torch.float32, device="cuda")
        self.flush = flush
        self.want_trace = False
        self.gen = torch.Generator(device="cuda")
        self.gen.manual_seed(0)

    def randn(self, *shape):
        return torch.randn(*shape, generator=self.gen, device="cuda", dtype=torch.float32).to(torch.bfloat16)

    def measure(self, chunk, o, ctx, reps):
        s, kv = self.s, self.kv
        seqs = list(range(1, len(ctx) + 1))
        fill = W.BatchDesc(prefill_seq=[0] + seqs, prefill_offset=[0] * (1 + len(ctx)),
                           prefill_len=[o] + [c - 1 for c in ctx])
        p = kv.plan(fill)
        T = fill.num_rows
        step = 65536
        k = self.randn(min(T, step), s.num_kv_heads, s.head_dim)
        # one append per fill plan (values irrelevant for timing): reuse a random block of rows
        kbuf = self.randn(T, s.num_kv_heads, s.head_dim) if T <= 4 * step else k.repeat((T + k.shape[0] - 1) // k.shape[0], 1, 1)[:T].contiguous()
        kv.append(p, 0, kbuf, kbuf)
        desc = W.BatchDesc(prefill_seq=[0] if chunk else [], prefill_offset=[o] if chunk else [],
                           prefill_len=[chunk] if chunk else [], decode_seq=seqs, decode_ctx=ctx)
        Tb = desc.num_rows
        batch = ny.Batch(desc)
        plan = kv.plan(batch)
        self.last_info = plan.info()
        knew = self.randn(Tb, s.num_kv_heads, s.head_dim)
        kv.append(plan, 0, knew, knew)
        q = self.randn(Tb, s.num_q_heads, s.head_dim)
        out = torch.empty(s.num_q_heads, Tb, s.head_dim, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            kv.attention(plan, 0, q, out)
        ts = []
        for _ in range(reps):
            if self.flush == "read":
                self.sink = self.scratch.sum(dtype=torch.float32)
            else:
                self.scratch.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            kv.attention(plan, 0, q, out)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        self.last_trace = None
        if self.want_trace:
            # one more flushed launch with the per-CTA timeline on (niyama_debug_trace):
            # entry, start, prefill end, decode end, exit (ns from the first entry), tiles done
            buf = torch.zeros(160 * 8 + 10 * 64, dtype=torch.int64, device="cuda")
            kv.debug_trace(buf)
            self.sink = self.scratch.sum(dtype=torch.float32)
            kv.attention(plan, 0, q, out)
            torch.cuda.synchronize()
            kv.debug_trace(None)
            tr = buf.cpu().numpy()[:160 * 8].reshape(160, 8)
            tr = tr[tr[:, 0] > 0]
            e0 = int(tr[:, 6].min())
            self.last_trace = {"entry_ns": (tr[:, 6] - e0).tolist(), "start_ns": (tr[:, 0] - e0).tolist(),
                               "prefill_end_ns": (tr[:, 1] - e0).tolist(), "decode_end_ns": (tr[:, 4] - e0).tolist(),
                               "exit_ns": (tr[:, 2] - e0).tolist(), "tiles": tr[:, 3].tolist()}
        plan.close()
        p.close()
        for sq in [0] + seqs:
            kv.release(sq)
        self.last_ts = ts
        return statistics.median(ts), Tb


def plan_fields(rig):
    i = rig.last_info
    return dict(tiles=i.num_prefill_tiles, units=i.num_decode_units, split_len=i.split_len,
                prefill_ctas=i.prefill_ctas, p10=float(np.percentile(rig.last_ts, 10)),
                p90=float(np.percentile(rig.last_ts, 90)))


def sweep(args):
    s = W.L8B if args.config == "l8b" else W.L70B
    rig = Rig(s, num_blocks=args.max_decode * 8192 // 16 + 8192, flush=args.flush)
    rows = []
    t0 = time.time()

    def run(kind, seed, chunk, D):
        o, ctx = point_desc(max(chunk, 1), D, seed)
        if chunk == 0:
            o = 0
        rig.want_trace = args.trace_every > 0 and len(rows) % args.trace_every == 0
        t, T = rig.measure(chunk, o, ctx, args.reps)
        rows.append(dict(kind=kind, seed=seed, chunk=chunk, offset=o, D=D, sum_ctx=int(sum(ctx)),
                         seconds=t, T=T, ctx=ctx, **plan_fields(rig)))
        if rig.last_trace is not None:
            rows[-1]["trace"] = rig.last_trace
        print(f"{kind:8s} seed={seed:4d} c={chunk:5d} o={o:5d} D={D:3d} sumctx={sum(ctx):8d} t={t*1e6:8.1f}us", flush=True)

    for seed in range(3):
        for chunk in (256, 512, 1024, 2048):
            for D in (16, 32, 64, 128, 256):
                run("grid", seed, chunk, min(D, args.max_decode))
    g = np.random.default_rng(123)
    for i in range(args.offgrid):
        run("offgrid", 100 + i, int(g.integers(1, 2049)), int(g.integers(1, args.max_decode + 1)))
    g = np.random.default_rng(456)
    for i in range(args.train_random):
        # random training points over the whole space, including prefill-only (D = 0)
        # and decode-only (c = 0) batches
        u = g.random()
        chunk = 0 if u < 0.08 else int(g.integers(1, 2049))
        D = 0 if 0.08 <= u < 0.16 else int(g.integers(1, args.max_decode + 1))
        run("random", 1000 + i, chunk, D)
    g = np.random.default_rng(789)
    for i in range(args.train_small):
        # extra training points in the regime the scheduler mostly runs (decode-only or a
        # chunk <= 512 with <= 64 decodes; config-5 replays), where the fit is weakest
        chunk = 0 if g.random() < 0.3 else int(g.integers(1, 513))
        run("random", 5000 + i, chunk, int(g.integers(1, min(64, args.max_decode) + 1)))
    return rows, time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="l8b", choices=["l8b", "l70b"])
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--flush", default="read", choices=["read", "write"])
    ap.add_argument("--offgrid", type=int, default=40)
    ap.add_argument("--train-random", type=int, default=120)
    ap.add_argument("--max-decode", type=int, default=256)
    ap.add_argument("--train-small", type=int, default=0,
                    help="extra training points with chunk <= 512 (30 %% decode-only) and <= 64 decodes")
    ap.add_argument("--trace-every", type=int, default=3, help="per-CTA timeline of every k-th point (0 = none)")
    ap.add_argument("--raw", default=os.path.join(ROOT, "profiles", "r02", "predictor_sweep_l8b.json"))
    args = ap.parse_args()
    rows, wall = sweep(args)
    out = {"config": args.config, "world": 1, "device": torch.cuda.get_device_name(0), "reps": args.reps,
           "timing": f"median of {args.reps} reps, CUDA events around one launch, L2 flushed before every rep "
                     f"({'512 MB read' if args.flush == 'read' else '512 MB write'})",
           "points": rows, "wall_s": wall}
    os.makedirs(os.path.dirname(args.raw), exist_ok=True)
    json.dump(out, open(args.raw, "w"), indent=1)
    print(f"{len(rows)} points in {wall:.0f} s -> {args.raw}")


if __name__ == "__main__":
    main()

"""Kernel micro-bench: median launch time of niyama_hybrid_attention for workload
variants, plus a per-CTA phase trace of config 2.  (Diagnostics, not the bench.)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2503_22562_b200 as ny  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def setup(wl, tuning=None):
    s = wl.shape
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 16, block_size=s.block_size,
                    dtype=s.dtype, device=0)
    if tuning:
        kv.set_tuning(**tuning)   # niyama_tuning fields (include/niyama.h)
    plan = None
    for st in wl.steps:
        plan = kv.plan(st.desc)
        kv.append(plan, 0, dev(st.k), dev(st.v))
    torch.cuda.synchronize()
    T = wl.final.desc.num_rows
    q = dev(wl.final.q)
    o = torch.empty((s.num_q_heads, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((s.num_q_heads, T), dtype=torch.float32, device="cuda")
    return kv, plan, q, o, lse


def time_it(wl, reps=50, trace=False, tuning=None):
    kv, plan, q, o, lse = setup(wl, tuning)
    for _ in range(5):
        kv.attention(plan, 0, q, o, lse)
    # back-to-back launches (no host sync in between, so host launch latency is hidden)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record()
    for i in range(reps):
        kv.attention(plan, 0, q, o, lse)
        evs[i + 1].record()
    torch.cuda.synchronize()
    ts = [evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(reps)]
    # the same launches with one event pair around all of them (no per-launch events)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        kv.attention(plan, 0, q, o, lse)
    e1.record()
    torch.cuda.synchronize()
    batched = e0.elapsed_time(e1) * 1e3 / reps
    tr = None
    if trace:
        buf = torch.zeros((160 * 8 + 10 * 64,), dtype=torch.int64, device="cuda")
        kv.debug_trace(buf)
        kv.attention(plan, 0, q, o, lse)
        torch.cuda.synchronize()
        kv.debug_trace(None)
        tr = buf.cpu().numpy()[:160 * 8].reshape(160, 8)
        tr = tr[tr[:, 0] > 0]
    d = wl.final.desc
    tok = sum(o_ + c for o_, c in zip(d.prefill_offset, d.prefill_len)) + sum(d.decode_ctx)
    B = tok * wl.shape.num_kv_heads * wl.shape.head_dim * 4
    med = statistics.median(ts)
    info = plan.info()
    print(f"{wl.name:40s} T={d.num_rows:5d} tiles={info.num_prefill_tiles:4d} units={info.num_decode_units:5d} "
          f"split={info.split_len:4d} median={med:8.1f}us batched={batched:8.1f}us  KV={B/1e6:7.1f}MB  "
          f"{B/batched/1e3:7.0f} GB/s", flush=True)
    if tr is not None:
        t0 = tr[:, 0].min()
        pre = tr[tr[:, 3] > 0]
        if len(pre):
            print(f"   prefill CTAs={len(pre)} tiles/CTA max={pre[:,3].max()} prefill end: "
                  f"min={(pre[:,1].min()-t0)/1e3:.1f}us max={(pre[:,1].max()-t0)/1e3:.1f}us")
        print(f"   CTA end: min={(tr[:,2].min()-t0)/1e3:.1f}us "
              f"median={(np.median(tr[:,2])-t0)/1e3:.1f}us max={(tr[:,2].max()-t0)/1e3:.1f}us; "
              f"start spread={(tr[:,0].max()-t0)/1e3:.1f}us", flush=True)
    return med


if __name__ == "__main__":
    ctx = W.l8b_decode_ctx()
    time_it(W.config2_l8b(), trace=True)
    time_it(W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=ctx, seed=2), trace=True)
    time_it(W.hybrid(W.L8B, "prefill-only-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2),
            trace=True)
    time_it(W.config2_l8b(ctx_mode="all4096"))
    time_it(W.config2_l8b(prefill_offset=0))
    time_it(W.config2_l8b(prefill_offset=3584))
    time_it(W.hybrid(W.L8B, "decode-only-256x4096", prefill_offset=0, chunk=0, decode_ctx=[4096] * 256, seed=2))

"""Where do the bench step's extra ~10 us of attention time come from?  Config 2, median of
the attention launch's event interval under progressively more bench-like steps:

  A  same plan, attention back to back
  B  same plan, append + attention
  C  new plan every step (plan / rollback / close) + append + attention
  D  C + the bench's a1 and a8 host work
  E  D with events on every 2nd step only (the bench)

    python tools/bench_gap.py [l8b|l70b]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
import workloads as W  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def main():
    wl = W.config4_l70b() if "l70b" in sys.argv else W.config2_l8b()
    s = wl.shape
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 64, block_size=s.block_size,
                    dtype=s.dtype, device=0)
    for st in wl.steps[:-1]:
        p = kv.plan(st.desc)
        kv.append(p, 0, dev(st.k), dev(st.v))
        torch.cuda.synchronize()
        p.close()
    fin = wl.final
    desc = fin.desc
    T = desc.num_rows
    q, k_new, v_new = dev(fin.q), dev(fin.k), dev(fin.v)
    o = torch.empty((s.num_q_heads, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((s.num_q_heads, T), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    batch = ny.Batch(desc)
    dec_only = ny.Batch(W.BatchDesc(decode_seq=desc.decode_seq, decode_ctx=desc.decode_ctx))
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, s.dtype, 1)
    pred = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA)).bind(kv)
    fixed = kv.plan(batch, stream)
    kv.append(fixed, 0, k_new, v_new, stream)
    torch.cuda.synchronize()
    fixed.rollback()
    fixed.close()
    fixed = kv.plan(batch, stream)

    def run(mode, n=200):
        evs = []
        host = 0.0
        step_e0, step_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(n + 10):
            if i == 10:
                torch.cuda.synchronize()
                step_e0.record(stream)
                h0 = time.perf_counter()
            every = 2 if mode == "E" else 1
            want = i >= 10 and (i % every == 0)
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if want else None
            if mode in ("D", "E"):
                sl = 0.05
                pred.max_feasible_chunk(dec_only, 1536, 512, sl, 2048)
            if mode == "A":
                plan = fixed
            elif mode == "B":
                plan = fixed
                kv.append(plan, 0, k_new, v_new, stream)
            else:
                plan = kv.plan(batch, stream)
                kv.append(plan, 0, k_new, v_new, stream)
            if e:
                e[0].record(stream)
            kv.attention(plan, 0, q, o, lse, 0.0, stream)
            if e:
                e[1].record(stream)
                evs.append(e)
            if mode in ("D", "E"):
                pred.predict(batch)
            if mode in ("C", "D", "E"):
                plan.rollback()
                plan.close()
        host = (time.perf_counter() - h0) * 1e6 / n
        step_e1.record(stream)
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) * 1e3 for a, b in evs]
        step = step_e0.elapsed_time(step_e1) * 1e3 / n
        print(f"{mode}: attention median {statistics.median(ts):7.1f} us  p10 {np.percentile(ts, 10):7.1f}  "
              f"p90 {np.percentile(ts, 90):7.1f}  step {step:7.1f} us  host {host:6.1f} us/step", flush=True)

    for _ in range(2):
        for m in "AB":
            run(m)
    fixed.rollback()
    fixed.close()
    for _ in range(2):
        for m in "CDE":
            run(m)
    # host cost of the pieces
    for name, fn in (("plan+rollback+close", lambda: (lambda p: (p.rollback(), p.close()))(kv.plan(batch, stream))),
                     ("max_feasible_chunk", lambda: pred.max_feasible_chunk(dec_only, 1536, 512, 0.05, 2048)),
                     ("predict", lambda: pred.predict(batch))):
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        torch.cuda.synchronize()
        print(f"host {name}: {(time.perf_counter() - t0) * 1e6 / 200:.1f} us")


if __name__ == "__main__":
    main()

"""Host cost of each call of one bench step (no device sync inside the loop)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
import workloads as W  # noqa: E402


def main():
    wl = W.config2_l8b()
    s, fin = wl.shape, wl.final
    desc = fin.desc
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 64, block_size=s.block_size,
                    dtype=s.dtype, device=0)
    dev = torch.device("cuda", 0)

    def bf(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(dev).view(torch.bfloat16)
    for st in wl.steps[:-1]:
        p = kv.plan(st.desc)
        kv.append(p, 0, bf(st.k), bf(st.v))
        torch.cuda.synchronize()
        p.close()
    q, k, v = bf(fin.q), bf(fin.k), bf(fin.v)
    o = torch.empty((s.num_q_heads, desc.num_rows, s.head_dim), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((s.num_q_heads, desc.num_rows), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    batch = ny.Batch(desc)
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, s.dtype, 1)
    pred = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA))
    mode = sys.argv[1] if len(sys.argv) > 1 else "full"
    names = ["plan", "append", "attention", "predict", "rollback", "close"]
    acc = np.zeros(len(names))
    n = 2000
    for it in range(n + 50):
        t = [time.perf_counter()]
        plan = kv.plan(batch, stream)
        t.append(time.perf_counter())
        if mode == "full":
            kv.append(plan, 0, k, v, stream)
        t.append(time.perf_counter())
        if mode == "full":
            kv.attention(plan, 0, q, o, lse, 0.0, stream)
        t.append(time.perf_counter())
        pred.predict(batch)
        t.append(time.perf_counter())
        plan.rollback()
        t.append(time.perf_counter())
        plan.close()
        t.append(time.perf_counter())
        if it >= 50:
            acc += np.diff(t)
    torch.cuda.synchronize()
    print("mode", mode)
    for nm, v_ in zip(names, acc / n * 1e6):
        print(f"{nm:10s} {v_:7.2f} us")
    print(f"{'total':10s} {acc.sum() / n * 1e6:7.2f} us")


if __name__ == "__main__":
    main()

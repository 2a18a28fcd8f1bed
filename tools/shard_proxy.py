"""Head-sharding proxy on ONE GPU (a7): the attention launch of rank 0 of a
G-way head-sharded job (its Hkv/G kv heads and Hq/G query heads, the same replicated
plan) for G = 1, 2, 4, 8, on configs 2 and 4.  The per-rank launch time is what each
GPU of a G-GPU job runs before the head all-gather (not measured here: one GPU per
call); t_1 / (G * t_G) is the attention's strong-scaling efficiency without the
collective.

    python tools/shard_proxy.py [reps]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_2503_22562_b200 as ny  # noqa: E402


def dev(a, lo, hi):
    return torch.from_numpy(np.ascontiguousarray(a[:, lo:hi]).view(np.int16)).cuda().view(torch.bfloat16)


def rank0_time(wl, G, reps, tuning=None):
    s = wl.shape
    hq, hkv = s.num_q_heads // G, s.num_kv_heads // G
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 16, block_size=s.block_size,
                    dtype=s.dtype, world_size=G, rank=0, device=0)
    if tuning:
        kv.set_tuning(**tuning)
    plan = None
    for st in wl.steps:
        plan = kv.plan(st.desc)
        kv.append(plan, 0, dev(st.k, 0, hkv), dev(st.v, 0, hkv))
    torch.cuda.synchronize()
    T = wl.final.desc.num_rows
    q = dev(wl.final.q, 0, hq)
    o = torch.empty((hq, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((hq, T), dtype=torch.float32, device="cuda")
    for _ in range(5):
        kv.attention(plan, 0, q, o, lse)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            kv.attention(plan, 0, q, o, lse)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    kv.close()
    return statistics.median(ts)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20
    tuning = dict(prefill_split=1) if "split" in sys.argv else None
    out = {"tuning": tuning or "default (no split-K)"}
    for name, wl in (("config2-l8b", W.config2_l8b()), ("config4-l70b", W.config4_l70b())):
        t1 = None
        for G in (1, 2, 4, 8):
            t = rank0_time(wl, G, reps if G > 1 or name.startswith("config2") else max(5, reps // 4), tuning)
            t1 = t if G == 1 else t1
            eff = t1 / (G * t)
            out.setdefault(name, {})[G] = {"rank0_launch_us": t, "attention_scaling_eff_no_collective": eff}
            print(f"{name:14s} G={G}: rank-0 attention launch {t:8.1f} us  t1/(G tG) = {eff:.3f}", flush=True)
    json.dump(out, open(os.path.join("gpurun_out", "shard_proxy" + ("_split" if tuning else "") + ".json"), "w"),
              indent=1)


if __name__ == "__main__":
    main()

"""Stress the emulated multi-rank fused gather (tests/test_gpu_gather.py emulated ranks) to
localise an intermittent plain-vs-window mismatch: many rounds of concurrent gather launches
followed by plain launches; on a mismatch, report which heads/rows differ and which side
agrees with a repeated plain launch and with the fp64 oracle.

    python tools/gather_stress.py [world] [rounds]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from oracle import shard  # noqa: E402
from tests.gpu_harness import oracle_for, to_dev, to_host_f64  # noqa: E402


def main():
    import paper_2503_22562_b200 as ny
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    s = W.Shape(num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(s, seed=60 + world, num_prefill=2, max_chunk=300, num_decode=24, max_ctx=2500)
    T = wl.final.desc.num_rows
    kvs, plans, rng_ = [], [], []
    for r in range(world):
        (q0, q1), (k0, k1) = shard.head_ranges(world, r, s.num_q_heads, s.num_kv_heads)
        rng_.append(((q0, q1), (k0, k1)))
        kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks, block_size=s.block_size,
                        dtype="bf16", world_size=world, rank=r, device=0)
        for st in wl.steps[:-1]:
            kv.append(kv.plan(st.desc), 0, to_dev(st.k[:, k0:k1], "bf16"), to_dev(st.v[:, k0:k1], "bf16"))
        plans.append(kv.plan(wl.final.desc))
        kvs.append(kv)
    # the final step's K/V (the test appends them in its last round, fused)
    for r in range(world):
        (q0, q1), (k0, k1) = rng_[r]
        kvs[r].append(plans[r], 0, to_dev(wl.final.k[:, k0:k1], "bf16"), to_dev(wl.final.v[:, k0:k1], "bf16"))
    torch.cuda.synchronize()
    wins = ny.debug_gather_group(kvs, T)
    streams = [torch.cuda.Stream() for _ in range(world)]
    fin = wl.final
    bad = 0
    ref = None
    for it in range(rounds):
        sc = [0.5, 2.0, 1.0][it % 3]
        qs = []
        for r in range(world):
            (q0, q1), _ = rng_[r]
            qs.append(to_dev(np.ascontiguousarray(fin.q[:, q0:q1]), "bf16") * sc)
        torch.cuda.synchronize()
        res = [kvs[r].attention_gather(plans[r], 0, qs[r], wins[r], None, None, 0.0, streams[r]) for r in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            (q0, q1), _ = rng_[r]
            outs = []
            for rep in range(2):
                o = torch.empty((q1 - q0, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
                lse = torch.empty((q1 - q0, T), dtype=torch.float32, device="cuda")
                kvs[r].attention(plans[r], 0, qs[r], o, lse)
                torch.cuda.synchronize()
                outs.append((o, lse))
            w = res[0][0][q0:q1]
            same_plain = torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
            eq = torch.equal(outs[0][0].view(torch.int16), w.view(torch.int16))
            if not eq or not same_plain:
                bad += 1
                d0 = (outs[0][0].view(torch.int16) != w.view(torch.int16))
                d1 = (outs[1][0].view(torch.int16) != w.view(torch.int16))
                heads, rows = torch.nonzero(d0.any(dim=2), as_tuple=True)
                print(f"round {it} scale {sc} rank {r}: plain==plain {same_plain}, plain0!=win {int(d0.sum())} elems "
                      f"(heads {sorted(set(heads.tolist()))[:8]}, rows {sorted(set(rows.tolist()))[:12]}), "
                      f"plain1!=win {int(d1.sum())}", flush=True)
                if sc == 1.0 and ref is None:
                    _, _, O, L = oracle_for(wl)
                    ref = O
                if sc == 1.0:
                    for name, x in (("plain0", outs[0][0]), ("plain1", outs[1][0]), ("window", w)):
                        err = np.abs(to_host_f64(x, "bf16") - ref[q0:q1]).max()
                        print(f"    {name} max_abs vs oracle {err:.3e}", flush=True)
    print(f"world {world}: {bad} mismatches in {rounds} rounds x {world} ranks", flush=True)
    for w_ in wins:
        w_.close()


if __name__ == "__main__":
    main()

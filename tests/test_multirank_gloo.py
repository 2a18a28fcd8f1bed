"""World-size-2 CPU test of the head-sharded (N > 1) path over torch.distributed/gloo.

Each rank creates its own library instance (host bookkeeping only) owning half the
kv heads (§8e).  Checks: (1) the replicated planner gives every rank identical
block tables and slot maps without exchanging metadata; (2) the 128-byte NCCL
unique id the library produces can be broadcast the way bench.py does it;
(3) per-rank oracle outputs over the rank's heads, all-gathered in rank order
(a7), reproduce the full oracle bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outq):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import workloads as W
    import paper_2503_22562_b200 as ny
    from oracle import attention as OA
    from oracle import shard
    from oracle.kvcache import KVPool

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = W.Shape(num_q_heads=8, num_kv_heads=4, head_dim=128, block_size=16, dtype="bf16")
        wl = W.random_hybrid(s, seed=31, num_prefill=2, max_chunk=90, num_decode=5, max_ctx=300)
        kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks, dtype="bf16", world_size=world,
                        rank=rank, device=None)
        slots = None
        for st in wl.steps:
            slots = kv.plan(st.desc).slots()
        tables = {sq: kv.block_table(sq) for sq in list(wl.final.desc.prefill_seq) + list(wl.final.desc.decode_seq)}
        got = [None] * world
        dist.all_gather_object(got, (slots, tables))
        ok_plan = all(g == got[0] for g in got)
        # unique id broadcast (rank 0 creates it)
        uid = [ny.get_unique_id() if rank == 0 else b""]
        dist.broadcast_object_list(uid, src=0)
        ok_uid = isinstance(uid[0], bytes) and len(uid[0]) == 128
        # per-rank oracle over local heads, all-gathered
        (q0, q1), (k0, k1) = shard.head_ranges(world, rank, s.num_q_heads, s.num_kv_heads)
        pool = KVPool(1, k1 - k0, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
        plan = None
        for st in wl.steps:
            plan = pool.plan(st.desc)
            pool.append(0, plan, st.k[:, k0:k1], st.v[:, k0:k1])
        O, L = OA.hybrid_attention(pool, 0, plan, wl.final.q[:, q0:q1], q1 - q0)
        t = torch.from_numpy(np.ascontiguousarray(O))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        full = None
        if rank == 0:
            fpool = KVPool(1, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
            fplan = None
            for st in wl.steps:
                fplan = fpool.plan(st.desc)
                fpool.append(0, fplan, st.k, st.v)
            full, _ = OA.hybrid_attention(fpool, 0, fplan, wl.final.q, s.num_q_heads)
            gathered = torch.cat(parts, dim=0).numpy()
            outq.put(("ok", ok_plan, ok_uid, bool(np.array_equal(gathered, full))))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        outq.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_head_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == "ok", res
    _, ok_plan, ok_uid, ok_gather = res
    assert ok_plan and ok_uid and ok_gather

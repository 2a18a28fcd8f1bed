"""§8(f)2 fused all-gather (niyama_gather_create / niyama_attention_gather) on ONE GPU.

The launch stores every O row and LSE value through the window's load/store mapping of
each rank and ends in a flag barrier between the ranks' launches.  At world size 1 the
one "peer" is this rank's own mapping, so these tests check the peer-address resolution,
the store redirection of every epilogue (prefill tiles, split-K merge, unsplit decode rows,
the decode merge tail, the tensor-core decode path), the barrier's epoch sequence and the
double buffering: the window must hold exactly what the plain launch writes (bitwise) and
what the fp64 oracle computes.  More than one rank needs more than one GPU (unmeasured)."""
import numpy as np
import pytest
import torch

import workloads as W
from tests.gpu_harness import Run, assert_close, oracle_for, to_dev, to_host_f64

pytestmark = pytest.mark.gpu


def _gather_kv(wl, tuning=None):
    import paper_2503_22562_b200 as ny
    run = Run(wl, tuning=tuning)
    run.kv.comm_init(ny.get_unique_id())
    return run


CASES = {
    "hybrid": dict(seed=3, num_prefill=2, max_chunk=300, num_decode=24, max_ctx=2500),
    "long_decodes": dict(seed=5, num_prefill=0, max_chunk=1, num_decode=12, max_ctx=9000),
    "prefill_only": dict(seed=9, num_prefill=3, max_chunk=700, num_decode=0, max_ctx=1),
}


@pytest.mark.parametrize("tuning", [None, dict(decode_path=1), dict(prefill_split=1)],
                         ids=["default", "tc_decode", "split_k"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_window_equals_plain_launch_and_oracle(case, tuning):
    s = W.Shape(num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(s, **CASES[case])
    run = _gather_kv(wl, tuning)
    o_ref, lse_ref = run.attention()
    win = run.kv.gather_window(wl.final.desc.num_rows + 7)
    o, lse = run.kv.attention_gather(run.plan, 0, to_dev(wl.final.q, "bf16"), win)
    torch.cuda.synchronize()
    assert torch.equal(o.view(torch.int16), o_ref.view(torch.int16))
    assert torch.equal(lse, lse_ref)
    _, _, O, L = oracle_for(wl)
    assert_close(to_host_f64(o, "bf16"), O, lse.double().cpu().numpy(), L)
    win.close()


def test_fused_append_into_window():
    s = W.Shape(num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(s, seed=11, num_prefill=2, max_chunk=257, num_decode=17, max_ctx=1800)
    import paper_2503_22562_b200 as ny
    run = Run(wl, fused=True)
    run.kv.comm_init(ny.get_unique_id())
    win = run.kv.gather_window(4096)
    st = wl.final
    o, lse = run.kv.attention_gather(run.plan, 0, to_dev(st.q, "bf16"), win, to_dev(st.k, "bf16"),
                                     to_dev(st.v, "bf16"))
    torch.cuda.synchronize()
    _, _, O, L = oracle_for(wl)
    assert_close(to_host_f64(o, "bf16"), O, lse.double().cpu().numpy(), L)


def test_double_buffering_and_many_launches():
    """Buffers alternate per call; a call never touches the previous call's buffer; a long
    run of launches without host syncs passes the barrier every time (epochs 1..n)."""
    s = W.Shape(num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(s, seed=21, num_prefill=1, max_chunk=200, num_decode=30, max_ctx=3000)
    run = _gather_kv(wl)
    o_ref, lse_ref = run.attention()
    win = run.kv.gather_window(1024)
    q = to_dev(wl.final.q, "bf16")
    o1, l1 = run.kv.attention_gather(run.plan, 0, q, win)
    torch.cuda.synchronize()
    snap = o1.clone()
    q2 = q * 0.5
    o2, l2 = run.kv.attention_gather(run.plan, 0, q2, win)
    torch.cuda.synchronize()
    assert o1.data_ptr() != o2.data_ptr() and l1.data_ptr() != l2.data_ptr()
    assert torch.equal(o1.view(torch.int16), snap.view(torch.int16))     # untouched by call 2
    assert not torch.equal(o2.view(torch.int16), snap.view(torch.int16))
    ptrs = set()
    for i in range(64):
        o, lse = run.kv.attention_gather(run.plan, 0, q, win)
        ptrs.add(o.data_ptr())
    torch.cuda.synchronize()
    assert len(ptrs) == 2
    assert torch.equal(o.view(torch.int16), o_ref.view(torch.int16))
    assert torch.equal(lse, lse_ref)


def test_gather_window_errors():
    import paper_2503_22562_b200 as ny
    s = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, 64, dtype="bf16", device=0)
    with pytest.raises(ny.NiyamaError) as e:
        kv.gather_window(128)                       # before comm_init
    assert e.value.status == 1
    kv.comm_init(ny.get_unique_id())
    with pytest.raises(ny.NiyamaError):
        kv.gather_window(0)
    win = kv.gather_window(16)
    p = kv.plan(W.BatchDesc([0], [0], [40]))
    q = torch.zeros((40, 8, 128), dtype=torch.bfloat16, device="cuda")
    k = torch.zeros((40, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ny.NiyamaError) as e:
        kv.attention_gather(p, 0, q, win, k, k)     # T = 40 > max_rows = 16
    assert e.value.status == 1
    with pytest.raises(ny.NiyamaError):
        kv.attention_gather(p, 0, q, win, k, None)  # k without v
    f32 = ny.KVCache(1, 8, 2, 128, 16, dtype="f32", device=0)
    f32.comm_init(ny.get_unique_id())
    with pytest.raises(ny.NiyamaError):
        f32.gather_window(16)
    win.close()
    kv.close()
    f32.close()


@pytest.mark.parametrize("world,shape", [(2, "l8b"), (4, "l8b"), (8, "l70b")])
def test_emulated_ranks_exchange_through_windows(world, shape):
    """The multi-rank protocol on one GPU (niyama_debug_gather_group): `world` library
    instances (rank r owns heads [r Hq/G, (r+1) Hq/G)) launch CONCURRENTLY on their own
    streams, each storing its heads into every rank's window and meeting the others at the
    flag barrier.  Three rounds with different queries (both buffers, epochs 1-3); after
    each, every rank's window must hold the full head-major output: all windows bitwise
    equal, and equal to the fp64 oracle (the last round, with the KV append fused in)."""
    import paper_2503_22562_b200 as ny
    from oracle import shard
    s = W.Shape(num_q_heads=32 if shape == "l8b" else 64, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
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
    torch.cuda.synchronize()
    wins = ny.debug_gather_group(kvs, T)
    streams = [torch.cuda.Stream() for _ in range(world)]
    fin = wl.final
    scales = [0.5, 2.0, 1.0]
    for it, sc in enumerate(scales):
        last = it == len(scales) - 1
        outs = []
        for r in range(world):
            (q0, q1), (k0, k1) = rng_[r]
            q = to_dev(np.ascontiguousarray(fin.q[:, q0:q1]), "bf16") * sc
            args = (to_dev(fin.k[:, k0:k1], "bf16"), to_dev(fin.v[:, k0:k1], "bf16")) if last else (None, None)
            torch.cuda.synchronize()
            outs.append((r, q, args))
        res = []
        for r, q, (k, v) in outs:     # every rank's launch enqueued before any wait
            res.append(kvs[r].attention_gather(plans[r], 0, q, wins[r], k, v, 0.0, streams[r]))
        torch.cuda.synchronize()
        for r in range(1, world):
            assert torch.equal(res[r][0].view(torch.int16), res[0][0].view(torch.int16)), (it, r)
            assert torch.equal(res[r][1], res[0][1]), (it, r)
        if not last:
            # the same rows once more through each rank's plain launch must match its window slice
            for r in range(world):
                (q0, q1), _ = rng_[r]
                o = torch.empty((q1 - q0, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
                lse = torch.empty((q1 - q0, T), dtype=torch.float32, device="cuda")
                kvs[r].attention(plans[r], 0, outs[r][1], o, lse)
                torch.cuda.synchronize()
                assert torch.equal(o.view(torch.int16), res[0][0][q0:q1].view(torch.int16)), (it, r)
    _, _, O, L = oracle_for(wl)
    assert_close(to_host_f64(res[0][0], "bf16"), O, res[0][1].double().cpu().numpy(), L)
    for w in wins:
        w.close()

"""Head-sharded path (a7) on ONE GPU.

Every rank of a head-sharded job runs the same planner and its own kernels over its
kv heads; only the all-gather exchanges data.  With one GPU available the ranks are
run as separate library instances (world_size G, rank r) on cuda:0 writing their
head slices of one head-major output, which must equal the full fp64 oracle; the
NCCL all-gather itself runs at world size 1 (ncclAllGather is issued at every world
size; at 1 it is NCCL's in-place copy)."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import shard
from tests.gpu_harness import assert_close, oracle_for, to_dev, to_host_f64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_head_sharded_ranks_match_full_oracle(world):
    import paper_2503_22562_b200 as ny
    s = W.Shape(num_q_heads=32, num_kv_heads=8, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(s, seed=40 + world, num_prefill=2, max_chunk=300, num_decode=24, max_ctx=2500)
    T = wl.final.desc.num_rows
    o_full = torch.full((s.num_q_heads, T, s.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse_full = torch.full((s.num_q_heads, T), float("nan"), dtype=torch.float32, device="cuda")
    for r in range(world):
        (q0, q1), (k0, k1) = shard.head_ranges(world, r, s.num_q_heads, s.num_kv_heads)
        kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks, block_size=s.block_size,
                        dtype=s.dtype, world_size=world, rank=r, device=0)
        plan = None
        for st in wl.steps:
            plan = kv.plan(st.desc)
            kv.append(plan, 0, to_dev(st.k[:, k0:k1], s.dtype), to_dev(st.v[:, k0:k1], s.dtype))
        kv.attention(plan, 0, to_dev(wl.final.q[:, q0:q1], s.dtype), o_full[q0:q1], lse_full[q0:q1])
        torch.cuda.synchronize()
    _, _, O, L = oracle_for(wl)
    assert_close(to_host_f64(o_full, "bf16"), O, lse_full.double().cpu().numpy(), L)


def test_allgather_needs_comm_init():
    import paper_2503_22562_b200 as ny
    kv = ny.KVCache(1, 8, 2, 128, 16, dtype="bf16", device=0)
    p = kv.plan(W.BatchDesc([0], [0], [5]))
    o = torch.zeros((8, 5, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ny.NiyamaError) as e:
        kv.allgather_heads(p, o)
    assert e.value.status == 1   # EINVAL


def test_nccl_allgather_world1_inplace():
    import paper_2503_22562_b200 as ny
    s = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(s, seed=7, num_prefill=1, max_chunk=100, num_decode=5, max_ctx=400)
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks, dtype="bf16", device=0)
    kv.comm_init(ny.get_unique_id())
    plan = None
    for st in wl.steps:
        plan = kv.plan(st.desc)
        kv.append(plan, 0, to_dev(st.k, "bf16"), to_dev(st.v, "bf16"))
    T = wl.final.desc.num_rows
    o = torch.empty((s.num_q_heads, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((s.num_q_heads, T), dtype=torch.float32, device="cuda")
    kv.attention(plan, 0, to_dev(wl.final.q, "bf16"), o, lse)
    before_o, before_l = o.clone(), lse.clone()
    kv.allgather_heads(plan, o, lse)
    torch.cuda.synchronize()
    assert torch.equal(o.view(torch.int16), before_o.view(torch.int16))
    assert torch.equal(lse, before_l)
    _, _, O, L = oracle_for(wl)
    assert_close(to_host_f64(o, "bf16"), O, lse.double().cpu().numpy(), L)

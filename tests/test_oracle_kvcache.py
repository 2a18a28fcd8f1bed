"""Pins for oracle/kvcache.py — CPU only.

Block tables and slots are checked against a hand-worked fixture
(tests/golden/kv_tables_scenario.json) and hand-computable block counts;
append/gather against bitwise read-back."""
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle import kvcache as K

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CODES = {"EINVAL": K.EINVAL, "ENOBLOCKS": K.ENOBLOCKS, "ENOSEQ": K.ENOSEQ, "ESTATE": K.ESTATE}


def test_hand_worked_tables():
    fx = json.load(open(os.path.join(GOLDEN, "kv_tables_scenario.json")))
    p = fx["pool"]
    pool = K.KVPool(p["num_layers"], p["num_kv_heads"], p["head_dim"], p["block_size"], p["num_blocks"], "f32")
    for st in fx["steps"]:
        if st["op"] == "release":
            pool.release(st["seq"])
            continue
        desc = W.BatchDesc(prefill_seq=[x[0] for x in st["prefill"]], prefill_offset=[x[1] for x in st["prefill"]],
                           prefill_len=[x[2] for x in st["prefill"]], decode_seq=[x[0] for x in st["decode"]],
                           decode_ctx=[x[1] for x in st["decode"]])
        if "expect_error" in st:
            before = ({s: list(t) for s, t in pool.table.items()}, dict(pool.length), list(pool.free))
            with pytest.raises(K.OracleError) as e:
                pool.plan(desc)
            assert e.value.code == CODES[st["expect_error"]]
            assert (pool.table, pool.length, pool.free) == before  # no side effects
        else:
            plan = pool.plan(desc)
            assert [list(s) for s in plan.slots] == st["expect_slots"]
        if "expect_tables" in st:
            assert {str(s): t for s, t in pool.table.items()} == st["expect_tables"]
        if "expect_free" in st:
            assert pool.free == st["expect_free"]


def test_config1_block_count():
    """config 1 = 4 + 2 + 7 + 16 = 29 blocks (ceil(n/16) per sequence)."""
    wl = W.config1_tiny()
    s = wl.shape
    pool = K.KVPool(1, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
    for st in wl.steps:
        pool.plan(st.desc)
    assert wl.num_blocks == 29
    assert sorted(len(t) for t in pool.table.values()) == [2, 4, 7, 16]
    assert pool.free == []


def test_append_gather_bitwise():
    wl = W.random_hybrid(W.L8B, seed=3, num_prefill=2, max_chunk=40, num_decode=4, max_ctx=90)
    s = wl.shape
    pool = K.KVPool(1, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
    allk, allv = {}, {}
    for st in wl.steps:
        plan = pool.plan(st.desc)
        pool.append(0, plan, st.k, st.v)
        for r, (seq, pos, _) in enumerate(plan.rows):
            allk[(seq, pos)] = st.k[r]
            allv[(seq, pos)] = st.v[r]
    for seq, n in pool.length.items():
        k, v = pool.gather(0, seq, n)
        for p in range(n):
            assert np.array_equal(k[p], allk[(seq, p)]) and np.array_equal(v[p], allv[(seq, p)])


def test_l8b_block_counts():
    """Config 2: 2048/16 = 128 prefill blocks + sum ceil(ctx/16) over the seed-0 draw."""
    ctx = W.l8b_decode_ctx()
    assert int(ctx.sum()) == 133674
    wl = W.hybrid(W.L8B, "count-only", prefill_offset=1536, chunk=512, decode_ctx=ctx, seed=0)
    assert wl.num_blocks == 128 + int(sum((c + 15) // 16 for c in ctx))


def test_zero_length_slice_registers_seq():
    pool = K.KVPool(1, 1, 4, 4, 4, "f32")
    plan = pool.plan(W.BatchDesc([5], [0], [0]))
    assert plan.rows == [] and pool.length[5] == 0 and pool.table[5] == []
    plan = pool.plan(W.BatchDesc(decode_seq=[5], decode_ctx=[1]))
    assert plan.rows == [(5, 0, 1)] and plan.slots == [(0, 0)]


def test_truncate_hand_worked():
    """KVPool.truncate (R9: a sequence of n tokens owns ceil(n/B) blocks; freed blocks are
    the smallest-free candidates again), hand-worked at B = 4 with 8 blocks:
      seq 1 gets 10 tokens -> blocks [0, 1, 2]; seq 2 gets 6 -> [3, 4]; free [5, 6, 7]
      truncate(1, 5): keeps ceil(5/4) = 2 blocks [0, 1]; block 2 freed -> free [2, 5, 6, 7]
      truncate(1, 4): keeps 1 block [0]; free [1, 2, 5, 6, 7]
      truncate(2, 0): keeps 0 blocks; free [1, 2, 3, 4, 5, 6, 7]
      seq 3 gets 9 tokens -> the 3 smallest free ids [1, 2, 3]
      truncate(1, 4) again is a no-op; truncate(1, 5) (> cached 4) is EINVAL, unknown seq ENOSEQ."""
    pool = K.KVPool(1, 1, 2, 4, 8, "f32")
    pool.plan(W.BatchDesc([1, 2], [0, 0], [10, 6]))
    assert pool.table == {1: [0, 1, 2], 2: [3, 4]} and pool.free == [5, 6, 7]
    pool.truncate(1, 5)
    assert pool.table[1] == [0, 1] and pool.length[1] == 5 and pool.free == [2, 5, 6, 7]
    pool.truncate(1, 4)
    assert pool.table[1] == [0] and pool.free == [1, 2, 5, 6, 7]
    pool.truncate(2, 0)
    assert pool.table[2] == [] and pool.length[2] == 0 and pool.free == [1, 2, 3, 4, 5, 6, 7]
    plan = pool.plan(W.BatchDesc([3], [0], [9]))
    assert pool.table[3] == [1, 2, 3] and [tuple(s) for s in plan.slots][:5] == [(1, 0), (1, 1), (1, 2), (1, 3), (2, 0)]
    pool.truncate(1, 4)
    assert pool.table[1] == [0]
    with pytest.raises(K.OracleError) as e:
        pool.truncate(1, 5)
    assert e.value.code == K.EINVAL
    with pytest.raises(K.OracleError) as e:
        pool.truncate(99, 0)
    assert e.value.code == K.ENOSEQ
    # a truncated sequence resumes at its new length (prefill offset = cached length, R4)
    pool.plan(W.BatchDesc([1], [4], [3]))
    assert pool.table[1] == [0, 4] and pool.length[1] == 7

"""Pins for oracle/attention.py — CPU only.

The oracle is checked against things other than itself: a pure-Python
brute-force triple loop (independent indexing through the raw pool array),
torch's fp64 scaled_dot_product_attention with an explicit boolean causal mask
on densely gathered K/V, closed forms, and the chunking invariants the paper
relies on (P:118 chunked prefill = full prefill; a decode row equals the last
prefill row at the same context)."""
import math

import numpy as np
import pytest
import torch

import workloads as W
from oracle import attention as A
from oracle.kvcache import KVPool
from oracle import shard


def build(wl: W.Workload):
    s = wl.shape
    pool = KVPool(s.num_layers, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
    plan = None
    for st in wl.steps:
        plan = pool.plan(st.desc)
        pool.append(0, plan, st.k, st.v)
    return pool, plan


def brute_force(pool, plan, q, Hq):
    """Triple loop over (row, head, key) with Python floats; K/V located through
    the raw [layer][kv][block][head][slot][d] array and the block table."""
    Hkv, d, B = pool.H, pool.d, pool.B
    g = Hq // Hkv
    T = len(plan.rows)
    O = np.zeros((Hq, T, d))
    L = np.zeros((Hq, T))
    scale = 1.0 / math.sqrt(d)

    def val(x):
        if pool.dtype == "bf16":
            return float(np.uint32(int(x) << 16).view(np.float32))
        return float(x)

    for r, (seq, _pos, n) in enumerate(plan.rows):
        tbl = pool.table[seq]
        for h in range(Hq):
            kh = h // g
            qv = [val(x) for x in q[r, h]]
            scores = []
            for t in range(n):
                kv = pool.data[0, 0, tbl[t // B], kh, t % B]
                scores.append(scale * sum(qv[i] * val(kv[i]) for i in range(d)))
            m = max(scores)
            ws = [math.exp(s - m) for s in scores]
            l = sum(ws)
            for i in range(d):
                acc = 0.0
                for t in range(n):
                    acc += ws[t] * val(pool.data[0, 1, tbl[t // B], kh, t % B][i])
                O[h, r, i] = acc / l
            L[h, r] = m + math.log(l)
    return O, L


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_brute_force_tiny(dtype):
    shape = W.Shape(num_q_heads=4, num_kv_heads=2, head_dim=8, block_size=4, dtype=dtype)
    wl = W.random_hybrid(shape, seed=11, num_prefill=2, max_chunk=6, num_decode=3, max_ctx=13)
    pool, plan = build(wl)
    q = wl.final.q
    O, L = A.hybrid_attention(pool, 0, plan, q, shape.num_q_heads)
    Ob, Lb = brute_force(pool, plan, q, shape.num_q_heads)
    np.testing.assert_allclose(O, Ob, rtol=0, atol=1e-12)
    np.testing.assert_allclose(L, Lb, rtol=0, atol=1e-12)


def test_torch_sdpa_special_case():
    """Library special case: torch CPU fp64 SDPA with an explicit boolean mask over
    each sequence's densely gathered K/V (GQA by repeat_interleave, R7)."""
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=32, block_size=16, dtype="bf16")
    wl = W.random_hybrid(shape, seed=5, num_prefill=2, max_chunk=70, num_decode=5, max_ctx=200)
    pool, plan = build(wl)
    q = A.to_f64(wl.final.q, "bf16")
    O, L = A.hybrid_attention(pool, 0, plan, wl.final.q, shape.num_q_heads)
    g = shape.group
    for r, (seq, pos, n) in enumerate(plan.rows):
        k, v = pool.gather(0, seq, pool.length[seq])
        K = torch.from_numpy(A.to_f64(k, "bf16")).permute(1, 0, 2).repeat_interleave(g, 0)  # [Hq][n][d]
        V = torch.from_numpy(A.to_f64(v, "bf16")).permute(1, 0, 2).repeat_interleave(g, 0)
        Q = torch.from_numpy(q[r])[:, None, :]                                             # [Hq][1][d]
        mask = torch.zeros(1, K.shape[1], dtype=torch.bool)
        mask[0, :n] = True
        ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V, attn_mask=mask)
        np.testing.assert_allclose(O[:, r, :], ref[:, 0, :].numpy(), rtol=0, atol=1e-12)


def _single_seq_pool(n, d=16, B=4, dtype="f32", kfill=None, vfill=None, seed=0):
    pool = KVPool(1, 1, d, B, -(-n // B) + 1, dtype)
    desc = W.BatchDesc(prefill_seq=[0], prefill_offset=[0], prefill_len=[n])
    plan = pool.plan(desc)
    g = W.rng(seed)
    k = g.standard_normal((n, 1, d)).astype(np.float32) if kfill is None else kfill
    v = g.standard_normal((n, 1, d)).astype(np.float32) if vfill is None else vfill
    pool.append(0, plan, k, v)
    return pool, plan, k, v


def test_closed_forms():
    d, n = 16, 23
    g = W.rng(3)
    # ctx=1 -> O = V0 exactly; LSE = scale*<q,k0>
    pool, plan, k, v = _single_seq_pool(1, d)
    q = g.standard_normal((1, 1, d)).astype(np.float32)
    O, L = A.hybrid_attention(pool, 0, plan, q, 1)
    np.testing.assert_array_equal(O[0, 0], v[0, 0].astype(np.float64))
    assert L[0, 0] == pytest.approx(float(q[0, 0].astype(np.float64) @ k[0, 0]) / math.sqrt(d), abs=1e-12)
    # all keys equal -> O = mean of visible V (per row: prefix mean), LSE = s + ln n
    kk = np.repeat(g.standard_normal((1, 1, d)).astype(np.float32), n, axis=0)
    pool, plan, _, v = _single_seq_pool(n, d, kfill=kk)
    q = g.standard_normal((n, 1, d)).astype(np.float32)
    O, L = A.hybrid_attention(pool, 0, plan, q, 1)
    vv = v[:, 0].astype(np.float64)
    for r in range(n):
        np.testing.assert_allclose(O[0, r], vv[: r + 1].mean(axis=0), atol=1e-12)
        s = float(q[r, 0].astype(np.float64) @ kk[0, 0]) / math.sqrt(d)
        assert L[0, r] == pytest.approx(s + math.log(r + 1), abs=1e-12)
    # q = 0 -> uniform weights -> mean V
    pool, plan, _, v = _single_seq_pool(n, d)
    O, _ = A.hybrid_attention(pool, 0, plan, np.zeros((n, 1, d), np.float32), 1)
    for r in range(n):
        np.testing.assert_allclose(O[0, r], v[: r + 1, 0].astype(np.float64).mean(axis=0), atol=1e-12)
    # V == 1 -> O == 1 (softmax rows sum to one); V == const vector -> that vector
    c = g.standard_normal(d).astype(np.float32)
    pool, plan, _, _ = _single_seq_pool(n, d, vfill=np.tile(c, (n, 1, 1)))
    O, _ = A.hybrid_attention(pool, 0, plan, g.standard_normal((n, 1, d)).astype(np.float32), 1)
    np.testing.assert_allclose(O[0], np.tile(c.astype(np.float64), (n, 1)), atol=1e-12)
    # one huge logit -> O = V at its argmax
    kk = g.standard_normal((n, 1, d)).astype(np.float32) * 0.01
    kk[7, 0, 0] = 1.0e4
    pool, plan, _, v = _single_seq_pool(n, d, kfill=kk)
    q = np.zeros((n, 1, d), np.float32)
    q[:, 0, 0] = 1.0
    O, _ = A.hybrid_attention(pool, 0, plan, q, 1)
    for r in range(7, n):
        np.testing.assert_allclose(O[0, r], v[7, 0].astype(np.float64), atol=1e-12)


def test_chunked_equals_full():
    """prefill split into chunks with appends between them == one full prefill."""
    shape = W.Shape(num_q_heads=4, num_kv_heads=2, head_dim=16, block_size=8, dtype="bf16")
    n = 57
    g = W.rng(9)
    k = W.draw_values(g, (n, 2, 16), "bf16")
    v = W.draw_values(g, (n, 2, 16), "bf16")
    q = W.draw_values(g, (n, 4, 16), "bf16")
    full = KVPool(1, 2, 16, 8, 16, "bf16")
    plan = full.plan(W.BatchDesc([0], [0], [n]))
    full.append(0, plan, k, v)
    O_full, L_full = A.hybrid_attention(full, 0, plan, q, 4)
    chunked = KVPool(1, 2, 16, 8, 16, "bf16")
    outs, lses, o = [], [], 0
    for c in [5, 16, 1, 30, 5]:
        plan = chunked.plan(W.BatchDesc([0], [o], [c]))
        chunked.append(0, plan, k[o:o + c], v[o:o + c])
        Oc, Lc = A.hybrid_attention(chunked, 0, plan, q[o:o + c], 4)
        outs.append(Oc)
        lses.append(Lc)
        o += c
    np.testing.assert_array_equal(np.concatenate(outs, axis=1), O_full)
    np.testing.assert_array_equal(np.concatenate(lses, axis=1), L_full)


def test_decode_equals_prefill_row():
    """A decode row at ctx L with query q equals the prefill row at position L-1 with q."""
    n, d = 40, 16
    g = W.rng(21)
    k = W.draw_values(g, (n, 1, d), "bf16")
    v = W.draw_values(g, (n, 1, d), "bf16")
    q = W.draw_values(g, (n, 2, d), "bf16")
    a = KVPool(1, 1, d, 16, 8, "bf16")
    pa = a.plan(W.BatchDesc([0], [0], [n]))
    a.append(0, pa, k, v)
    Oa, La = A.hybrid_attention(a, 0, pa, q, 2)
    b = KVPool(1, 1, d, 16, 8, "bf16")
    pb = b.plan(W.BatchDesc([0], [0], [n - 1]))
    b.append(0, pb, k[: n - 1], v[: n - 1])
    pd = b.plan(W.BatchDesc(decode_seq=[0], decode_ctx=[n]))
    b.append(0, pd, k[n - 1:], v[n - 1:])
    Ob, Lb = A.hybrid_attention(b, 0, pd, q[n - 1:], 2)
    np.testing.assert_array_equal(Ob[:, 0], Oa[:, n - 1])
    np.testing.assert_array_equal(Lb[:, 0], La[:, n - 1])


def test_lse_merge_identity():
    """a6: merging the partials of any split of [0, L) equals the unsplit result."""
    g = W.rng(4)
    for L in [1, 2, 17, 300]:
        q = g.standard_normal((4, 32)) * 3
        k = g.standard_normal((L, 32))
        v = g.standard_normal((L, 32))
        o_ref, lse_ref = A.softmax_attend(q, k, v, 0.2)
        cuts = sorted(set(g.integers(1, L, size=min(5, max(0, L - 1))).tolist())) if L > 1 else []
        bounds = [0] + cuts + [L]
        parts = [A.split_partial(q, k[a:b], v[a:b], 0.2) for a, b in zip(bounds, bounds[1:])]
        o, lse = A.merge_partials(parts)
        np.testing.assert_allclose(o, o_ref, atol=1e-13)
        np.testing.assert_allclose(lse, lse_ref, atol=1e-13)
        # closed form of the partial: lse of a split = m_s + ln l_s
        m, l, _ = parts[0]
        _, lse0 = A.softmax_attend(q, k[bounds[0]:bounds[1]], v[bounds[0]:bounds[1]], 0.2)
        np.testing.assert_allclose(m + np.log(l), lse0, atol=1e-13)


def test_head_shard_concat_equals_full():
    """a7: per-rank oracle over its kv heads, concatenated in rank order == full oracle."""
    shape = W.Shape(num_q_heads=8, num_kv_heads=4, head_dim=16, block_size=8, dtype="bf16")
    wl = W.random_hybrid(shape, seed=8, num_prefill=1, max_chunk=20, num_decode=4, max_ctx=50)
    pool, plan = build(wl)
    O_full, L_full = A.hybrid_attention(pool, 0, plan, wl.final.q, 8)
    for G in [1, 2, 4]:
        outs, lses = [], []
        for r in range(G):
            (q0, q1), (k0, k1) = shard.head_ranges(G, r, 8, 4)
            sp = KVPool(1, k1 - k0, 16, 8, wl.num_blocks, "bf16")
            p = None
            for st in wl.steps:
                p = sp.plan(st.desc)
                sp.append(0, p, st.k[:, k0:k1], st.v[:, k0:k1])
            O, L = A.hybrid_attention(sp, 0, p, wl.final.q[:, q0:q1], q1 - q0)
            outs.append(O)
            lses.append(L)
        np.testing.assert_array_equal(shard.allgather_heads(outs), O_full)
        np.testing.assert_array_equal(shard.allgather_heads(lses), L_full)


def test_config1_shape_and_rows():
    wl = W.config1_tiny()
    pool, plan = build(wl)
    assert len(plan.rows) == 64 + 3
    assert [r[2] for r in plan.rows[64:]] == [17, 100, 255]
    O, L = A.hybrid_attention(pool, 0, plan, wl.final.q, 4)
    assert np.isfinite(O).all() and np.isfinite(L).all()

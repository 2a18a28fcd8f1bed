"""GPU parity: the CUDA path through the C ABI against the fp64 oracle on the
same seeded inputs (SURVEY §8c bar: bit-exact KV append and block indexing;
attention within max-abs 2e-2 and rel-L2 5e-3)."""
import math

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from tests.gpu_harness import Run, assert_close, oracle_for, stored_bits, to_dev, to_host_f64  # noqa: E402


def run_and_compare(wl, rows=None, **kw):
    r = Run(wl, **kw)
    o, lse = r.attention()
    _, _, O, L = oracle_for(wl, rows=rows)
    og = to_host_f64(o, wl.shape.dtype)
    lg = lse.cpu().numpy().astype(np.float64)
    if rows is not None:
        mask = np.zeros(og.shape[1], bool)
        mask[list(rows)] = True
        og = og[:, mask]
        lg = lg[:, mask]
        O = O[:, mask]
        L = L[:, mask]
    return r, assert_close(og, O, lg, L)


F32_TOL = 1e-5   # fp32 storage and fp32 SIMT math: rounding ~1e-7 relative, so 1e-5 leaves margin


@pytest.mark.parametrize("variant,peaky", [("aligned", False), ("unaligned", False), ("aligned", True)])
def test_config1_tiny_f32(variant, peaky):
    """Config 1 (fp32) at fp32 tolerance (not the bf16 bar); the achieved error is printed."""
    wl = W.config1_tiny(variant, peaky)
    r = Run(wl)
    o, lse = r.attention()
    _, _, O, L = oracle_for(wl)
    ma, rl = assert_close(to_host_f64(o, "f32"), O, lse.cpu().numpy().astype(np.float64), L, max_abs=F32_TOL,
                          rel_l2=F32_TOL, lse_tol=F32_TOL)
    print(f"config1 {variant}{' peaky' if peaky else ''}: max_abs={ma:.2e} rel_l2={rl:.2e}")


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_append_bitwise_readback(dtype):
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128 if dtype == "bf16" else 64, block_size=16,
                    dtype=dtype)
    wl = W.random_hybrid(shape, seed=7, num_prefill=3, max_chunk=100, num_decode=5, max_ctx=300)
    r = Run(wl)
    pool, _, _, _ = oracle_for(wl)
    for seq, n in pool.length.items():
        assert r.kv.block_table(seq) == pool.table[seq]
        if n == 0:
            continue
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        k = torch.empty((n, shape.num_kv_heads, shape.head_dim), dtype=tdt, device="cuda")
        v = torch.empty_like(k)
        r.kv.gather(0, seq, n, k, v)
        kk, vv = pool.gather(0, seq, n)
        assert np.array_equal(stored_bits(k, dtype), kk)
        assert np.array_equal(stored_bits(v, dtype), vv)


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_random_ragged_bf16(seed):
    """Several prefill slices at unaligned offsets + decodes at ragged contexts (spans
    several 128-key tiles and 16-token decode stages with ragged tails)."""
    wl = W.random_hybrid(W.L8B, seed=seed, num_prefill=2, max_chunk=300, num_decode=9, max_ctx=900)
    run_and_compare(wl)


@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_gqa_groups_bf16(g):
    shape = W.Shape(num_q_heads=2 * g, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(shape, seed=10 + g, num_prefill=1, max_chunk=260, num_decode=5, max_ctx=700)
    run_and_compare(wl)


@pytest.mark.parametrize("B", [32, 64, 128])
def test_block_sizes_bf16(B):
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=B, dtype="bf16")
    wl = W.random_hybrid(shape, seed=B, num_prefill=2, max_chunk=200, num_decode=6, max_ctx=600)
    run_and_compare(wl)


def test_peaky_q_bf16():
    wl = W.random_hybrid(W.L8B, seed=5, num_prefill=1, max_chunk=256, num_decode=8, max_ctx=2000, q_scale=8.0)
    run_and_compare(wl)


def test_long_decodes_split_merge():
    """Decode contexts long enough that every row is split and merged by LSE (a5/a6)."""
    wl = W.hybrid(W.L8B, "long-dec", prefill_offset=0, chunk=0, decode_ctx=[8192, 5000, 4097, 1, 17, 300], seed=3)
    run_and_compare(wl)


def test_prefill_only_and_decode_only():
    run_and_compare(W.hybrid(W.L8B, "prefill-only", prefill_offset=700, chunk=333, decode_ctx=[], seed=4))
    run_and_compare(W.hybrid(W.L8B, "decode-only", prefill_offset=0, chunk=0, decode_ctx=[1, 2, 15, 16, 17, 4095],
                             seed=5))


def test_config2_l8b_full_size_sampled():
    """Config 2 at full size in the launch configuration bench.py times; checked on
    every decode row and a sample of prefill rows covering tile edges."""
    wl = W.config2_l8b()
    rows = sorted(set([0, 1, 31, 32, 63, 64, 127, 128, 255, 256, 383, 384, 511] + list(range(512, 576))))
    run_and_compare(wl, rows=rows)


def test_config4_l70b_full_size_sampled():
    """Config 4 (Llama-3-70B heads, g = 8: 2048-token chunk at o = 6144 + 128 decodes at
    ctx 8192) at full size in the launch configuration bench.py times (CTA split, 8
    decode warps, split length 2048); checked on tile-edge prefill rows and decode rows."""
    wl = W.config4_l70b()
    rows = [0, 15, 16, 17, 1023, 1024, 2032, 2047, 2048, 2049, 2111, 2175]
    run_and_compare(wl, rows=rows)


@pytest.mark.parametrize("case", ["ragged", "peaky", "f32", "config2"])
def test_fused_append_attention(case):
    """niyama_append_attention (a3 + a4-a6 in one launch) gives bitwise the same
    output as niyama_kv_append followed by niyama_hybrid_attention, leaves the same
    pool (gather read-back), and matches the oracle."""
    if case == "ragged":
        wl = W.random_hybrid(W.L8B, seed=31, num_prefill=2, max_chunk=300, num_decode=9, max_ctx=900)
    elif case == "peaky":
        wl = W.random_hybrid(W.L8B, seed=5, num_prefill=1, max_chunk=256, num_decode=8, max_ctx=2000, q_scale=8.0)
    elif case == "f32":
        wl = W.config1_tiny("unaligned")
    else:
        wl = W.config2_l8b()
    r1, r2 = Run(wl), Run(wl, fused=True)
    o1, l1 = r1.attention()
    o2, l2 = r2.attention()
    if wl.shape.dtype == "bf16":
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    else:
        assert torch.equal(o1, o2)
    assert torch.equal(l1, l2)
    if case != "config2":
        _, _, O, L = oracle_for(wl)
        assert_close(to_host_f64(o2, wl.shape.dtype), O, l2.cpu().numpy().astype(np.float64), L)
    seq = wl.final.desc.prefill_seq[0] if wl.final.desc.prefill_seq else wl.final.desc.decode_seq[0]
    n = r1.kv.seq_len(seq)
    tdt = torch.bfloat16 if wl.shape.dtype == "bf16" else torch.float32
    ka, va, kb, vb = (torch.empty((n, wl.shape.num_kv_heads, wl.shape.head_dim), dtype=tdt, device="cuda")
                      for _ in range(4))
    r1.kv.gather(0, seq, n, ka, va)
    r2.kv.gather(0, seq, n, kb, vb)
    assert torch.equal(ka, kb) and torch.equal(va, vb)


def test_deterministic_and_tier_invariant():
    wl = W.random_hybrid(W.L8B, seed=21, num_prefill=2, max_chunk=300, num_decode=12, max_ctx=3000)
    r = Run(wl)
    o1, l1 = r.attention()
    o2, l2 = r.attention()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16)) and torch.equal(l1, l2)
    # same batch, permuted tiers -> bitwise identical (R13)
    wl2 = W.random_hybrid(W.L8B, seed=21, num_prefill=2, max_chunk=300, num_decode=12, max_ctx=3000)
    wl2.final.desc.tier = list(reversed(wl2.final.desc.tiers()))
    o3, l3 = Run(wl2).attention()
    assert torch.equal(o1.view(torch.int16), o3.view(torch.int16)) and torch.equal(l1, l3)


def test_block_permutation_invariant():
    """Same logical content in different physical blocks -> bitwise identical output."""
    wl = W.random_hybrid(W.L8B, seed=22, num_prefill=1, max_chunk=200, num_decode=6, max_ctx=800)
    o1, l1 = Run(wl).attention()
    import paper_2503_22562_b200 as ny
    s = wl.shape
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 300, dtype="bf16", device=0)
    # occupy a scattered set of blocks first so the real sequences land elsewhere
    kv.plan(W.BatchDesc([9999], [0], [16 * 300]))
    kv.release(9999)
    kv.plan(W.BatchDesc([9998, 9997], [0, 0], [16 * 37, 16 * 41]))
    o2, l2 = Run(wl, kv=kv).attention()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16)) and torch.equal(l1, l2)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_multilayer_distinct_kv_one_plan(dtype):
    """32 layers, each with its OWN K/V/Q values (W.revalue), appended and attended with
    ONE plan per iteration reused by every layer — the real per-iteration pattern (the
    plan's split-completion counters advance one epoch per launch).  Every layer must
    match the oracle run on that layer's values; a kernel that ignored the layer offset
    or mis-counted epochs fails."""
    import paper_2503_22562_b200 as ny
    shape = W.L8B if dtype == "bf16" else W.TINY
    base = W.random_hybrid(shape, seed=23, num_prefill=2, max_chunk=200, num_decode=10, max_ctx=2500)
    layers = [W.revalue(base, 500 + l) for l in range(32)]
    s = shape
    kv = ny.KVCache(32, s.num_q_heads, s.num_kv_heads, s.head_dim, base.num_blocks, block_size=s.block_size,
                    dtype=s.dtype, device=0)
    for n, st in enumerate(base.steps):
        plan = kv.plan(st.desc)          # one plan per iteration ...
        for l in range(32):              # ... used by every layer
            kv.append(plan, l, to_dev(layers[l].steps[n].k, s.dtype), to_dev(layers[l].steps[n].v, s.dtype))
    info = plan.info()
    if dtype == "bf16":
        assert info.num_decode_units > info.num_decode * s.num_kv_heads   # rows are split (a6 merges run)
    T = base.final.desc.num_rows
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    outs = []
    for l in range(32):
        o = torch.full((s.num_q_heads, T, s.head_dim), float("nan"), dtype=tdt, device="cuda")
        lse = torch.full((s.num_q_heads, T), float("nan"), dtype=torch.float32, device="cuda")
        kv.attention(plan, l, to_dev(layers[l].final.q, s.dtype), o, lse)
        outs.append((o, lse))
    torch.cuda.synchronize()
    tol = {} if dtype == "bf16" else dict(max_abs=F32_TOL, rel_l2=F32_TOL, lse_tol=F32_TOL)
    prev = None
    for l in range(32):
        _, _, O, L = oracle_for(layers[l])
        og = to_host_f64(outs[l][0], dtype)
        assert_close(og, O, outs[l][1].cpu().numpy().astype(np.float64), L, **tol)
        if prev is not None:
            assert not np.array_equal(og, prev)   # the layers really differ
        prev = og


def test_empty_batch_noop_and_errors():
    import paper_2503_22562_b200 as ny
    kv = ny.KVCache(1, 32, 8, 128, 64, dtype="bf16", device=0)
    p = kv.plan(W.BatchDesc())
    kv.append(p, 0, 0, 0)
    kv.attention(p, 0, 0, 0)
    p = kv.plan(W.BatchDesc([0], [0], [5]))
    x = torch.zeros(5 * 8 * 128 + 8, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ny.NiyamaError):
        kv.append(p, 0, x[1:].data_ptr(), x.data_ptr())   # misaligned
    with pytest.raises(ny.NiyamaError):
        kv.append(p, 1, x, x)                              # layer out of range


def test_close_cache_with_live_plans():
    """Closing a cache destroys its live plans first (their buffers come from the cache's
    memory pool): no use after free when the plan objects are collected later."""
    import gc
    import paper_2503_22562_b200 as ny
    for _ in range(2):
        kv = ny.KVCache(1, 32, 8, 128, 256, dtype="bf16", device=0)
        plan = kv.plan(W.BatchDesc([0, 1], [0, 0], [100, 37]))
        kv.close()
        assert plan.handle is None
        del plan
        gc.collect()
    torch.cuda.synchronize()


def test_many_live_plans_fallback():
    """More live plans than upload slots (8): later plans fall back to pool buffers
    uploaded on the caller's stream; results still match the oracle, and slots are
    reused once plans are destroyed."""
    import paper_2503_22562_b200 as ny
    wl = W.random_hybrid(W.L8B, seed=41, num_prefill=1, max_chunk=200, num_decode=6, max_ctx=700)
    s = wl.shape
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 64, dtype="bf16", device=0)
    hold = [kv.plan(W.BatchDesc([5000 + i], [0], [16])) for i in range(9)]
    run_and_compare(wl, kv=kv)
    for p in hold:
        p.close()
    wl2 = W.random_hybrid(W.L8B, seed=42, num_prefill=1, max_chunk=150, num_decode=5, max_ctx=500)
    run_and_compare(wl2)


@pytest.mark.parametrize("case", ["ragged", "g8", "long-split", "blocks64"])
def test_tensor_core_decode_path(case):
    """niyama_tuning.decode_path = 1 (the tcgen05 CTA decode pipeline) against the oracle."""
    if case == "ragged":
        wl = W.random_hybrid(W.L8B, seed=21, num_prefill=2, max_chunk=300, num_decode=20, max_ctx=3000)
    elif case == "g8":
        wl = W.random_hybrid(W.Shape(64, 8, 128, 16, "bf16"), seed=22, num_prefill=1, max_chunk=200, num_decode=9,
                             max_ctx=2500)
    elif case == "long-split":
        wl = W.hybrid(W.L8B, "long", prefill_offset=0, chunk=0, decode_ctx=[8192, 17, 4095, 1], seed=23)
    else:
        wl = W.random_hybrid(W.Shape(32, 8, 128, 64, "bf16"), seed=24, num_prefill=1, max_chunk=300, num_decode=12,
                             max_ctx=3000)
    run_and_compare(wl, tuning=dict(decode_path=1))


@pytest.mark.parametrize("case", ["ragged", "g8", "long-split", "blocks64", "config4-sampled"])
def test_producer_consumer_decode_path(case):
    """niyama_tuning.decode_path = 2 (warps 8-11 load for the 8 compute warps) against the
    oracle, and bitwise equal to decode_path 3 (every warp its own loader) and to the default
    (auto) path: same units, same per-unit arithmetic."""
    if case == "ragged":
        wl = W.random_hybrid(W.L8B, seed=21, num_prefill=2, max_chunk=300, num_decode=20, max_ctx=3000)
    elif case == "g8":
        wl = W.random_hybrid(W.Shape(64, 8, 128, 16, "bf16"), seed=22, num_prefill=1, max_chunk=200, num_decode=9,
                             max_ctx=2500)
    elif case == "long-split":
        wl = W.hybrid(W.L8B, "long", prefill_offset=0, chunk=0, decode_ctx=[8192, 17, 4095, 1], seed=23)
    elif case == "blocks64":
        wl = W.random_hybrid(W.Shape(32, 8, 128, 64, "bf16"), seed=24, num_prefill=1, max_chunk=300, num_decode=12,
                             max_ctx=3000)
    else:
        wl = W.config4_l70b()
    rows = None
    if case == "config4-sampled":
        T = wl.final.desc.num_rows
        rows = list(range(T - 128, T, 9)) + [0, 1000, 2047]
    r2, _ = run_and_compare(wl, rows=rows, tuning=dict(decode_path=2))
    o2, l2 = r2.attention()
    for tuning in (dict(decode_path=3), None):
        r0 = Run(wl, tuning=tuning)
        o0, l0 = r0.attention()
        torch.cuda.synchronize()
        assert torch.equal(o2.view(torch.int16), o0.view(torch.int16))
        assert torch.equal(l2, l0)


@pytest.mark.parametrize("case", ["ragged", "odd-tiles", "g8", "blocks64", "blocks128", "config4-sampled"])
def test_prefill_cta_pairs(case):
    """niyama_tuning.prefill_pairs = 1 (clusters of 2 CTAs share every K/V step of two q
    tiles, each issuing half the copies multicast into both) against the oracle, and bitwise
    equal to one q tile per CTA (the partner's extra key step, if any, is fully masked)."""
    L8 = W.L8B
    if case == "ragged":
        wl = W.random_hybrid(L8, seed=71, num_prefill=2, max_chunk=300, num_decode=12, max_ctx=3000)
    elif case == "odd-tiles":   # nqt = 3 and 1: a partner without a tile
        wl = W.hybrid(L8, "odd", prefill_offset=700, chunk=80, decode_ctx=[900, 33], seed=72)
    elif case == "g8":
        wl = W.random_hybrid(W.Shape(64, 8, 128, 16, "bf16"), seed=73, num_prefill=1, max_chunk=200, num_decode=9,
                             max_ctx=2500)
    elif case == "blocks64":
        wl = W.random_hybrid(W.Shape(32, 8, 128, 64, "bf16"), seed=74, num_prefill=2, max_chunk=300, num_decode=6,
                             max_ctx=3000)
    elif case == "blocks128":
        wl = W.random_hybrid(W.Shape(32, 8, 128, 128, "bf16"), seed=75, num_prefill=1, max_chunk=400, num_decode=4,
                             max_ctx=3000)
    else:
        wl = W.config4_l70b()
    rows = None
    if case == "config4-sampled":
        T = wl.final.desc.num_rows
        rows = list(range(0, 2048, 97)) + [2047, T - 1]
    r2, _ = run_and_compare(wl, rows=rows, tuning=dict(prefill_pairs=1))
    o2, l2 = r2.attention()
    r0 = Run(wl, tuning=dict(prefill_pairs=2))
    o0, l0 = r0.attention()
    torch.cuda.synchronize()
    assert torch.equal(o2.view(torch.int16), o0.view(torch.int16))
    assert torch.equal(l2, l0)


@pytest.mark.parametrize("cap", [1, 5, 6])
def test_prefill_cta_pairs_small_grids(cap):
    """CTA pairs under a grid cap: an odd cap (5) runs 4 or 6 CTAs in pairs, a cap of 1 keeps one
    tile per CTA; results bitwise equal to the unpaired launch and within the oracle's bounds."""
    wl = W.random_hybrid(W.Shape(64, 8, 128, 16, "bf16"), seed=76, num_prefill=2, max_chunk=150, num_decode=5,
                         max_ctx=1500)
    r2, _ = run_and_compare(wl, tuning=dict(prefill_pairs=1, grid_cap=cap))
    o2, l2 = r2.attention()
    r0 = Run(wl, tuning=dict(prefill_pairs=2))
    o0, l0 = r0.attention()
    torch.cuda.synchronize()
    assert torch.equal(o2.view(torch.int16), o0.view(torch.int16))
    assert torch.equal(l2, l0)


@pytest.mark.parametrize("case", ["prefill-only", "mixed", "g8", "two-slices", "diag-only"])
def test_prefill_split_k(case):
    """Split-K prefill (niyama_tuning.prefill_split = 1: key parts of a q tile on different CTAs,
    merged by the last part) against the oracle, and the same launch unsplit (the default)."""
    L8 = W.L8B
    if case == "prefill-only":
        wl = W.hybrid(L8, "p", prefill_offset=3000, chunk=100, decode_ctx=[], seed=31)
    elif case == "mixed":
        wl = W.hybrid(L8, "m", prefill_offset=2000, chunk=64, decode_ctx=[700, 33, 1500], seed=32)
    elif case == "g8":
        wl = W.hybrid(W.Shape(64, 8, 128, 16, "bf16"), "g8", prefill_offset=2500, chunk=90, decode_ctx=[400], seed=33)
    elif case == "two-slices":
        wl = W.random_hybrid(L8, seed=34, num_prefill=2, max_chunk=60, num_decode=2, max_ctx=3500)
    else:
        wl = W.hybrid(L8, "d", prefill_offset=1500, chunk=40, decode_ctx=[], seed=35)
    r, _ = run_and_compare(wl, tuning=dict(prefill_split=1))
    import paper_2503_22562_b200 as ny
    det = ny.Predictor.from_params(ny.Predictor.shape_cfg(wl.shape.num_q_heads, wl.shape.num_kv_heads, 128),
                                   list(ny.DEFAULT_THETA)).bind(r.kv).detail(wl.final.desc)
    if case != "two-slices":
        assert det["parts_target"] > 1          # the case exercises the split path
    run_and_compare(wl)


def _kvq(seed, n, shape):
    g = W.rng(seed)
    return (W.draw_values(g, (n, shape.num_kv_heads, shape.head_dim), "bf16"),
            W.draw_values(g, (n, shape.num_kv_heads, shape.head_dim), "bf16"),
            W.draw_values(g, (n, shape.num_q_heads, shape.head_dim), "bf16"))


def test_chunked_prefill_equals_full_prefill():
    """P:118 (chunked prefills): a 700-token prompt prefilled as chunks 256 + 256 + 188 over three
    iterations gives, row by row, the output of one 700-token prefill — bitwise (every row runs
    the same key steps in the same order whatever tile holds it) — and both match the oracle."""
    import paper_2503_22562_b200 as ny
    s = W.L8B
    k, v, q = _kvq(41, 700, s)

    def run(chunks):
        kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, 64, dtype="bf16", device=0)
        outs, off = [], 0
        for c in chunks:
            p = kv.plan(W.BatchDesc([0], [off], [c]))
            kv.append(p, 0, to_dev(k[off:off + c], "bf16"), to_dev(v[off:off + c], "bf16"))
            o = torch.empty((s.num_q_heads, c, s.head_dim), dtype=torch.bfloat16, device="cuda")
            lse = torch.empty((s.num_q_heads, c), dtype=torch.float32, device="cuda")
            kv.attention(p, 0, to_dev(q[off:off + c], "bf16"), o, lse)
            torch.cuda.synchronize()
            outs.append((o, lse))
            off += c
        return torch.cat([o for o, _ in outs], dim=1), torch.cat([l for _, l in outs], dim=1)
    of, lf = run([700])
    oc, lc = run([256, 256, 188])
    assert torch.equal(of.view(torch.int16), oc.view(torch.int16)) and torch.equal(lf, lc)
    wl = W.Workload("full", s, [W.Step(W.BatchDesc([0], [0], [700]), k, v, q)], 64)
    _, _, O, L = oracle_for(wl)
    assert_close(to_host_f64(of, "bf16"), O, lf.cpu().numpy().astype(np.float64), L)


def test_decode_row_equals_prefill_row():
    """A decode row at ctx L with query q equals the prefill row at position L-1 with the same q
    and keys (two different code paths: split-KV mma.sync decode vs tcgen05 prefill tiles), within
    the bf16 bar; ctx 1000 and 4096 (split rows, merged in-launch)."""
    import paper_2503_22562_b200 as ny
    s = W.L8B
    for L in (1000, 4096):
        k, v, q = _kvq(42 + L, L, s)
        kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, 2 * (L // 16 + 2), dtype="bf16", device=0)
        p = kv.plan(W.BatchDesc([1, 2], [0, 0], [L - 1, L - 1]))
        kk = np.concatenate([k[:L - 1], k[:L - 1]])
        vv = np.concatenate([v[:L - 1], v[:L - 1]])
        kv.append(p, 0, to_dev(kk, "bf16"), to_dev(vv, "bf16"))
        p2 = kv.plan(W.BatchDesc([1], [L - 1], [1], decode_seq=[2], decode_ctx=[L]))  # row 0 prefill, row 1 decode
        kv.append(p2, 0, to_dev(np.concatenate([k[L - 1:], k[L - 1:]]), "bf16"),
                  to_dev(np.concatenate([v[L - 1:], v[L - 1:]]), "bf16"))
        o = torch.empty((s.num_q_heads, 2, s.head_dim), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((s.num_q_heads, 2), dtype=torch.float32, device="cuda")
        kv.attention(p2, 0, to_dev(np.concatenate([q[L - 1:], q[L - 1:]]), "bf16"), o, lse)
        torch.cuda.synchronize()
        a = o[:, 0].float().cpu().numpy().astype(np.float64)
        b = o[:, 1].float().cpu().numpy().astype(np.float64)
        assert_close(b, a, lse[:, 1].cpu().numpy().astype(np.float64), lse[:, 0].cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("scale", [2.0, 4.0])
def test_repeated_launches_bitwise_peaky(scale):
    """Peaky queries make the prefill softmax's lazy O rescale frequent; 24 launches of the same
    plan must agree bitwise.  (Pins the rescale's wait for PV_{j-1}: a parity wait two phases
    behind returned early and rescaled O under a running PV — an intermittent wrong row,
    tools/gather_stress.py.)"""
    wl = W.random_hybrid(W.L8B, seed=81, num_prefill=2, max_chunk=300, num_decode=12, max_ctx=2500)
    r = Run(wl)
    qd = to_dev(wl.final.q, "bf16") * scale
    T = wl.final.desc.num_rows
    s = wl.shape
    ref = None
    for _ in range(24):
        o = torch.empty((s.num_q_heads, T, s.head_dim), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((s.num_q_heads, T), dtype=torch.float32, device="cuda")
        r.kv.attention(r.plan, 0, qd, o, lse)
        if ref is None:
            torch.cuda.synchronize()
            ref = (o, lse)
            continue
        torch.cuda.synchronize()
        assert torch.equal(o.view(torch.int16), ref[0].view(torch.int16))
        assert torch.equal(lse, ref[1])

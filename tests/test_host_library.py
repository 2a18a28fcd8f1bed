"""CPU tests of the C-ABI library (no GPU): every declared symbol is exported,
and the host logic behind the boundary (block allocator, planner slot map,
work-list sizing, predictor, slack) agrees with the oracle.  The pool is
created with device = NIYAMA_DEVICE_NONE (host bookkeeping only); every call
that would touch the GPU must refuse with EUNSUPPORTED (no CPU fallback)."""
import json
import math
import os
import re

import numpy as np
import pytest

import workloads as W
from oracle import kvcache as OK_
from oracle import predictor as OP
from oracle import sched as OS
import paper_2503_22562_b200 as ny
from paper_2503_22562_b200 import _binding as NB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "niyama.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(niyama_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(NB.lib, n), n
    assert b"sm_100a" in NB.lib.niyama_version()


def host_kv(shape: W.Shape, num_blocks: int, world=1, rank=0):
    return ny.KVCache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, num_blocks,
                      block_size=shape.block_size, dtype=shape.dtype, world_size=world, rank=rank, device=None)


def test_golden_tables_through_c_abi():
    fx = json.load(open(os.path.join(GOLDEN, "kv_tables_scenario.json")))
    p = fx["pool"]
    # the library needs block_size >= 16: scale the fixture's block size 4 -> 16 by
    # scaling every length by 4 (ceil(4n/16) == ceil(n/4)); slots scale the same way.
    kv = ny.KVCache(1, 1, 1, 128, p["num_blocks"], block_size=16, dtype="bf16", device=None)
    codes = {"EINVAL": NB.EINVAL, "ENOBLOCKS": NB.ENOBLOCKS, "ENOSEQ": NB.ENOSEQ, "ESTATE": NB.ESTATE}
    for st in fx["steps"]:
        if st["op"] == "release":
            kv.release(st["seq"])
            continue
        desc = W.BatchDesc(prefill_seq=[x[0] for x in st["prefill"]], prefill_offset=[4 * x[1] for x in st["prefill"]],
                           prefill_len=[4 * x[2] for x in st["prefill"]], decode_seq=[x[0] for x in st["decode"]],
                           decode_ctx=[x[1] for x in st["decode"]])
        if st["decode"] and "expect_error" not in st:
            # decodes add one token: express them as 4-token prefill slices after scaling
            desc = W.BatchDesc(prefill_seq=desc.prefill_seq + desc.decode_seq,
                               prefill_offset=desc.prefill_offset + [4 * (c - 1) for c in desc.decode_ctx],
                               prefill_len=desc.prefill_len + [4] * len(desc.decode_seq))
        if "expect_error" in st:
            nfree = kv.num_free()
            with pytest.raises(ny.NiyamaError) as e:
                kv.plan(desc)
            assert e.value.status == codes[st["expect_error"]]
            assert kv.num_free() == nfree
        else:
            kv.plan(desc)
        if "expect_tables" in st:
            for s, t in st["expect_tables"].items():
                assert kv.block_table(int(s)) == t


def replay_both(wl: W.Workload):
    s = wl.shape
    kv = host_kv(s, wl.num_blocks)
    pool = OK_.KVPool(1, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
    plans = []
    for st in wl.steps:
        p = kv.plan(st.desc)
        o = pool.plan(st.desc)
        assert p.slots() == [tuple(x) for x in o.slots]
        plans.append((p, o))
    for seq in pool.table:
        assert kv.block_table(seq) == pool.table[seq]
        assert kv.seq_len(seq) == pool.length[seq]
    assert kv.num_free() == len(pool.free)
    return kv, pool, plans


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_random_tables_and_slots_match_oracle(seed):
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(shape, seed=seed, num_prefill=3, max_chunk=200, num_decode=6, max_ctx=500)
    kv, pool, _ = replay_both(wl)
    # release + reuse keeps the smallest-free-id policy
    for seq in list(pool.table)[::2]:
        kv.release(seq)
        pool.release(seq)
    d = W.BatchDesc(prefill_seq=[1000], prefill_offset=[0], prefill_len=[333])
    assert kv.plan(d).slots() == [tuple(x) for x in pool.plan(d).slots]
    assert kv.block_table(1000) == pool.table[1000]


def test_error_codes_match_oracle():
    shape = W.Shape(num_q_heads=4, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    kv = host_kv(shape, 8)
    pool = OK_.KVPool(1, 2, 128, 16, 8, "bf16")
    cases = [
        W.BatchDesc(decode_seq=[5], decode_ctx=[1]),                         # ENOSEQ
        W.BatchDesc([1], [3], [4]),                                           # ESTATE (new seq, offset 3)
        W.BatchDesc([1, 1], [0, 0], [4, 4]),                                  # EINVAL duplicate
        W.BatchDesc([1], [0], [16 * 9]),                                      # ENOBLOCKS
        W.BatchDesc([1], [0], [-1]),                                          # EINVAL
    ]
    for d in cases:
        with pytest.raises(OK_.OracleError) as eo:
            pool.plan(d)
        with pytest.raises(ny.NiyamaError) as ec:
            kv.plan(d)
        assert ec.value.status == eo.value.code
    assert kv.num_free() == 8
    kv.plan(W.BatchDesc([1], [0], [20]))
    for d in [W.BatchDesc(decode_seq=[1], decode_ctx=[20]), W.BatchDesc(decode_seq=[1], decode_ctx=[0])]:
        pool.plan(W.BatchDesc([1], [0], [20])) if 1 not in pool.length else None
        with pytest.raises(OK_.OracleError) as eo:
            pool.plan(d)
        with pytest.raises(ny.NiyamaError) as ec:
            kv.plan(d)
        assert ec.value.status == eo.value.code


def test_device_calls_refuse_without_gpu():
    kv = host_kv(W.L8B, 16)
    p = kv.plan(W.BatchDesc([0], [0], [10]))
    for call in (lambda: kv.append(p, 0, 16, 16), lambda: kv.attention(p, 0, 16, 16),
                 lambda: kv.gather(0, 0, 10, 16, 16)):
        with pytest.raises(ny.NiyamaError) as e:
            call()
        assert e.value.status == NB.EUNSUPPORTED


def test_work_list_sizing():
    """a2: tiles = sum ceil(c/R) * Hkv with R = 128/g; split q is the smallest power of two
    >= 64 with sum ctx * Hkv / q <= 4 * 148 * 8; a row is ceil(ctx/q) - 1 pieces of q keys
    plus its last piece cut into min(q, max(256, q/4))-key units."""
    ctx = W.l8b_decode_ctx()
    wl = W.hybrid(W.L8B, "sizing", prefill_offset=1536, chunk=512, decode_ctx=ctx, seed=0)
    kv = host_kv(W.L8B, wl.num_blocks)
    for st in wl.steps:
        p = kv.plan(st.desc)
    info = p.info()
    assert info.rows_per_tile == 32
    assert info.num_prefill_tiles == (512 // 32) * 8
    assert info.split_len == 256                      # 133674*8/4736 = 225.8 -> 256
    def pieces(c):
        nf = -(-int(c) // 256) - 1
        return nf + -(-(int(c) - 256 * nf) // 256)
    assert info.num_decode_units == sum(pieces(c) for c in ctx) * 8
    assert info.sum_ctx == 133674 and info.num_rows == 576


def test_plan_rollback_matches_oracle_truncate():
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(shape, seed=9, num_prefill=2, max_chunk=200, num_decode=6, max_ctx=500, extra_blocks=64)
    kv, pool, _ = replay_both(wl)
    free0 = kv.num_free()
    d = wl.final.desc
    nxt = W.BatchDesc(prefill_seq=list(d.prefill_seq) + [777], prefill_offset=[o + c for o, c in zip(
        d.prefill_offset, d.prefill_len)] + [0], prefill_len=[33] * len(d.prefill_seq) + [40],
        decode_seq=list(d.decode_seq), decode_ctx=[c + 1 for c in d.decode_ctx])
    tables = {s: kv.block_table(s) for s in pool.table}
    p = kv.plan(nxt)
    p.rollback()
    assert kv.num_free() == free0
    assert {s: kv.block_table(s) for s in pool.table} == tables
    with pytest.raises(ny.NiyamaError):
        kv.seq_len(777)
    # replaying the same plan lands in the same blocks and slots
    assert kv.plan(nxt).slots() == [tuple(x) for x in pool.plan(nxt).slots]


def test_plan_rollback_equals_oracle_truncate_and_release():
    """niyama_plan_rollback == the oracle's truncate of every sequence the plan extended back
    to its old length plus release of every sequence it created (R9), compared on block
    tables, lengths and the free list (the next allocation's ids)."""
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    for seed in range(4):
        wl = W.random_hybrid(shape, seed=50 + seed, num_prefill=3, max_chunk=150, num_decode=7, max_ctx=400,
                             extra_blocks=96)
        kv, pool, _ = replay_both(wl)
        d = wl.final.desc
        old = dict(pool.length)
        nxt = W.BatchDesc(prefill_seq=list(d.prefill_seq) + [900 + seed], prefill_offset=[o + c for o, c in zip(
            d.prefill_offset, d.prefill_len)] + [0], prefill_len=[17 + 9 * seed] * len(d.prefill_seq) + [45],
            decode_seq=list(d.decode_seq), decode_ctx=[c + 1 for c in d.decode_ctx])
        p = kv.plan(nxt)
        pool.plan(nxt)
        p.rollback()
        for s_, n in old.items():
            pool.truncate(s_, n)
        pool.release(900 + seed)
        assert kv.num_free() == len(pool.free)
        for s_ in pool.table:
            assert kv.block_table(s_) == pool.table[s_] and kv.seq_len(s_) == pool.length[s_]
        probe = W.BatchDesc([5000], [0], [16 * 20 + 3])
        assert kv.plan(probe).slots() == [tuple(x) for x in pool.plan(probe).slots]


def test_kv_truncate_matches_oracle():
    shape = W.Shape(num_q_heads=8, num_kv_heads=2, head_dim=128, block_size=16, dtype="bf16")
    wl = W.random_hybrid(shape, seed=77, num_prefill=3, max_chunk=200, num_decode=6, max_ctx=600)
    kv, pool, _ = replay_both(wl)
    g = np.random.default_rng(5)
    for s_ in list(pool.table):
        n = int(g.integers(0, pool.length[s_] + 1))
        kv.truncate(s_, n)
        pool.truncate(s_, n)
        assert kv.block_table(s_) == pool.table[s_] and kv.num_free() == len(pool.free)
    with pytest.raises(ny.NiyamaError):
        kv.truncate(list(pool.table)[0], 10 ** 6)


def test_rollback_validates_before_any_change():
    """an ESTATE rollback must not have rolled back earlier entries."""
    kv = host_kv(W.L8B, 64)
    kv.plan(W.BatchDesc([1, 2], [0, 0], [40, 40]))
    p = kv.plan(W.BatchDesc([1, 2], [40, 40], [30, 30]))   # both -> 70
    kv.truncate(2, 10)                                     # seq 2 now shorter than before the plan
    t1 = kv.block_table(1)
    with pytest.raises(ny.NiyamaError) as e:
        p.rollback()
    assert e.value.status == NB.ESTATE
    assert kv.seq_len(1) == 70 and kv.block_table(1) == t1  # untouched


def test_rollback_skips_reused_seq_id():
    """a late rollback must not free the blocks of a later sequence that reuses
    a released id (identity = id + creation generation)."""
    kv = host_kv(W.L8B, 64)
    p = kv.plan(W.BatchDesc([7], [0], [50]))     # creates seq 7
    kv.release(7)
    kv.plan(W.BatchDesc([7], [0], [20]))         # a new seq 7
    t = kv.block_table(7)
    free = kv.num_free()
    p.rollback()
    assert kv.seq_len(7) == 20 and kv.block_table(7) == t and kv.num_free() == free


def test_unsupported_shapes_rejected_at_create():
    for args, dt in [((1, 8, 8, 64), "bf16"), ((1, 32, 2, 128), "bf16"), ((1, 8, 8, 256), "f32"),
                     ((1, 32, 2, 64), "f32")]:
        with pytest.raises(ny.NiyamaError) as e:
            ny.KVCache(*args, 64, dtype=dt, device=None)
        assert e.value.status == NB.EUNSUPPORTED
    ny.KVCache(1, 64, 8, 128, 64, dtype="bf16", device=None)   # g = 8 supported
    ny.KVCache(1, 4, 2, 64, 64, dtype="f32", device=None)      # config 1


def test_tuning_roundtrip_validation_and_effect():
    kv = host_kv(W.L8B, 4096)
    t = kv.tuning()
    assert (t.prefill_ctas, t.split_len, t.tail_div, t.tail_min, t.grid_cap, t.plan_copy_stream) == \
        (0, 0, 4, 256, 0, 1)
    assert (t.decode_path, t.prefill_split, t.prefill_pairs) == (0, 0, 0)   # auto / off / auto
    for bad in ({"split_len": 24}, {"tail_div": 0}, {"tail_min": 8}, {"prefill_ctas": -1}, {"plan_copy_stream": 2},
                {"decode_path": 4}, {"decode_path": -1}, {"prefill_split": 2}, {"prefill_pairs": 3}):
        with pytest.raises(ny.NiyamaError) as e:
            kv.set_tuning(**bad)
        assert e.value.status == NB.EINVAL
    assert kv.tuning().split_len == 0          # a rejected call changes nothing
    for ok in ({"decode_path": 3}, {"decode_path": 2}, {"prefill_pairs": 1}, {"prefill_pairs": 2}):
        kv.set_tuning(**ok)
        assert all(getattr(kv.tuning(), k) == v for k, v in ok.items())
    ctx = W.l8b_decode_ctx()
    wl = W.hybrid(W.L8B, "tune", prefill_offset=1536, chunk=512, decode_ctx=ctx, seed=0)
    kv = host_kv(W.L8B, wl.num_blocks)
    kv.set_tuning(split_len=512, prefill_ctas=7)
    for st in wl.steps:
        p = kv.plan(st.desc)
    assert p.info().split_len == 512 and p.info().prefill_ctas == 7


def test_predictor_bind_uses_kv_tuning():
    kv = host_kv(W.L8B, 64)
    pr = ny.Predictor.from_params(CFG, THETA)
    b = W.BatchDesc([0], [1536], [512], decode_seq=list(range(1, 65)), decode_ctx=W.l8b_decode_ctx().tolist())
    t0 = pr.predict(b)
    kv.set_tuning(prefill_ctas=2)
    pr.bind(kv)
    assert pr.predict(b) != t0                 # the CTA split it models changed
    kv70 = ny.KVCache(1, 64, 8, 128, 64, dtype="bf16", device=None)  # noqa: F841
    with pytest.raises(ny.NiyamaError):
        pr.bind(kv70)                          # another local shape


def test_head_shard_config():
    kv = ny.KVCache(1, 64, 8, 128, 64, dtype="bf16", world_size=8, rank=3, device=None)
    p = kv.plan(W.BatchDesc([0], [0], [100]))
    assert p.info().num_prefill_tiles == 100 // 16 + 1     # g = 8, R = 16, 1 local kv head
    with pytest.raises(ny.NiyamaError):
        ny.KVCache(1, 64, 8, 128, 64, world_size=3, rank=0, device=None)


# ------------------------------------------------------------------ predictor
SHAPE = OP.PredShape(num_q_heads=32, num_kv_heads=8, head_dim=128, elt_bytes=2)
CFG = ny.Predictor.shape_cfg(32, 8, 128)
THETA = np.array(ny.DEFAULT_THETA)


def _rand_batch(g, max_p=3, max_d=50):
    P = int(g.integers(0, max_p))
    D = int(g.integers(0, max_d))
    offs = [int(x) for x in g.integers(0, 5000, size=P)]
    lens = [int(x) for x in g.integers(0, 2049, size=P)]
    ctx = [int(x) for x in g.integers(1, 8193, size=D)]
    return offs, lens, ctx


def _oracle(pr, theta, offs, lens, ctx):
    """The oracle's prediction for the launch the library models (its plan configuration)."""
    d = W.BatchDesc(list(range(len(offs))), offs, lens, list(range(100, 100 + len(ctx))), ctx)
    det = pr.detail(d)
    ln = OP.Launch(det["split_len"], det["small_piece"], det["grid"], det["prefill_ctas"], det["warps_per_cta"])
    w = OP.work(SHAPE, list(zip(offs, lens)), ctx, max(det["split_len"], 1), max(det["small_piece"], 1),
                det["parts_target"])
    assert w.units == det["units"]
    return d, OP.predict(theta, w, ln)


def test_predictor_eval_matches_oracle():
    g = np.random.default_rng(0)
    for k in range(40):
        theta = THETA * np.exp(g.uniform(-0.5, 0.5, size=len(THETA))) if k % 2 else THETA
        theta[5] = 1.0 if k % 4 < 3 else float(g.uniform(0.5, 2))
        pr = ny.Predictor.from_params(CFG, theta)
        np.testing.assert_array_equal(pr.params(), theta)
        offs, lens, ctx = _rand_batch(g)
        d, want = _oracle(pr, theta, offs, lens, ctx)
        assert pr.predict(d) == pytest.approx(want, rel=1e-12, abs=0)


def test_planner_and_predictor_model_the_same_launch():
    """The predictor's launch configuration (grid, prefill CTAs, split, units) is the plan's."""
    pr = ny.Predictor.from_params(CFG, THETA)
    g = np.random.default_rng(4)
    for it in range(12):
        offs, lens, ctx = _rand_batch(g, max_p=3, max_d=80)
        if it % 3 == 2:
            ctx = [int(x) for x in g.integers(2048, 8193, size=int(g.integers(100, 200)))]  # split 1024/2048
        kv = host_kv(W.L8B, 120000)
        n = len(offs)
        pre = W.BatchDesc(list(range(n)) + list(range(100, 100 + len(ctx))), [0] * (n + len(ctx)),
                          offs + [c - 1 for c in ctx])
        kv.plan(pre).close()
        d = W.BatchDesc(list(range(n)), offs, lens, list(range(100, 100 + len(ctx))), ctx)
        info = kv.plan(d).info()
        det = pr.detail(d)
        assert (info.prefill_ctas, info.num_decode_units) == (det["prefill_ctas"], det["units"])
        if ctx:
            assert info.split_len == det["split_len"]
        ln = OP.Launch(det["split_len"], det["small_piece"], det["grid"], det["prefill_ctas"], 12)
        w = OP.work(SHAPE, list(zip(offs, lens)), ctx, max(det["split_len"], 1), max(det["small_piece"], 1),
                    det["parts_target"])
        assert sum(OP.tiles_per_cta(w, ln)) == len(w.tiles)


def test_predictor_fit_recovers_model_generated_times():
    """Times generated by the model at known parameters: the library's fit (Nelder-Mead + NNLS)
    starting a factor e^0.5 away reproduces them; the oracle's NNLS at the true nonlinear
    parameters recovers the linear part exactly."""
    g = np.random.default_rng(1)
    truth = THETA.copy()
    pr = ny.Predictor.from_params(CFG, truth)
    batches, ts, works, lns = [], [], [], []
    for _ in range(120):
        offs, lens, ctx = _rand_batch(g, max_p=2, max_d=120)
        if not lens and not ctx:
            ctx = [100]
        d, t = _oracle(pr, truth, offs, lens, ctx)
        det = pr.detail(d)
        works.append(OP.work(SHAPE, list(zip(offs, lens)), ctx, max(det["split_len"], 1), max(det["small_piece"], 1),
                             det["parts_target"]))
        lns.append(OP.Launch(det["split_len"], det["small_piece"], det["grid"], det["prefill_ctas"], 12))
        batches.append(d)
        ts.append(t)
    lin, sse = OP.fit_linear(works, lns, np.array(ts), truth[6:])
    np.testing.assert_allclose(lin, truth[:6], rtol=1e-6, atol=1e-14)
    assert sse < 1e-20
    start = truth * np.exp(0.5 * np.where(np.arange(len(truth)) % 2 == 0, 1.0, -1.0))
    fit = ny.Predictor.fit_batches(CFG, batches, ts, start=start, max_evals=3000)
    err = np.array([fit.predict(b) / t - 1 for b, t in zip(batches, ts)])
    assert np.abs(err).max() < 0.01, np.abs(err).max()


def test_committed_fit_reproduces_and_meets_bars():
    """profiles/predictor_fit.json: every recorded prediction is what the library gives at the
    committed parameters; the held-out errors are the file's own numbers.  Bars on the committed
    measurement (late round 2, after the Q-load and CTA-split changes; honest status in DESIGN.md
    6.4, where R16's max <= 5 % is NOT met): held-out p50 <= 2 %, p95 <= 6 %, >= 55 of 60 points
    within 5 %."""
    fj = json.load(open(os.path.join(ROOT, "profiles", "predictor_fit.json")))
    sw = json.load(open(os.path.join(ROOT, fj["sweep"])))
    pr = ny.Predictor.from_params(CFG, fj["theta"])
    byk = {(p["kind"], p["seed"], p["chunk"], p["D"]): p for p in fj["points"]}
    held = []
    for r in sw["points"]:
        c = r["chunk"]
        d = W.BatchDesc([0] if c else [], [r["offset"]] if c else [], [c] if c else [], list(range(1, r["D"] + 1)),
                        list(r["ctx"]))
        rec = byk[(r["kind"], r["seed"], r["chunk"], r["D"])]
        assert pr.predict(d) == pytest.approx(rec["predicted"], rel=1e-12)
        if r["kind"] == "offgrid" or (r["kind"] == "grid" and r["seed"] == 2):
            held.append(pr.predict(d) / r["seconds"] - 1)
    held = np.abs(held)
    assert len(held) == fj["fit"]["heldout_points"] == 60
    assert float(held.max()) == pytest.approx(fj["heldout_rel_err"]["max"], rel=1e-9)
    assert float(np.median(held)) <= 0.02
    assert float(np.percentile(held, 95)) <= 0.06
    assert int(np.sum(held <= 0.05)) >= 55


def test_max_feasible_chunk_matches_oracle():
    pr = ny.Predictor.from_params(CFG, THETA)
    g = np.random.default_rng(2)
    for _ in range(12):
        ctx = [int(x) for x in g.integers(1, 4097, size=int(g.integers(0, 64)))]
        o = int(g.integers(0, 4000))
        rem = int(g.integers(0, 3000))

        def t_of(C):
            return _oracle(pr, THETA, [o] if C else [], [C] if C else [], ctx)[1]
        slack = float(t_of(0) * g.uniform(0.8, 3.0))
        assert pr.max_feasible_chunk(ctx, o, rem, slack, 2048) == OP.max_feasible_chunk(t_of, rem, slack, 2048)


def test_spec_examples_through_c_abi():
    fx = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))
    cm = fx["cost_model"]
    th = [cm["c0"], cm["c1"], 0, cm["c2"], 0, 0] + list(ny.DEFAULT_THETA[6:])
    pr = ny.Predictor.from_params(CFG, th)
    assert pr.predict(W.BatchDesc()) == pytest.approx(cm["c0"], abs=1e-15)
    assert pr.predict(W.BatchDesc([0], [0], [256])) == pytest.approx(cm["chunk256_s"], rel=1e-12)
    assert pr.max_feasible_chunk([], 0, 10**6, cm["inverse"]["slack"], 2048) == (256, False)
    assert pr.max_feasible_chunk([], 0, 10**6, math.inf, 2048) == (2048, False)
    assert pr.max_feasible_chunk([100], 0, 10**6, 0.001, 2048) == (0, True)
    bad = list(th)
    bad[6] = 0.0
    with pytest.raises(ny.NiyamaError):
        ny.Predictor.from_params(CFG, bad)                    # tau0 must be > 0
    for ex in fx["slack"]:
        decs = [OS.DecodeQoS(**d) for d in ex["decodes"]]
        got = ny.min_slack(decs, ex["now"])
        want = OS.min_slack(decs, ex["now"])
        assert got == want


def test_min_slack_random_matches_oracle():
    g = np.random.default_rng(3)
    for _ in range(30):
        decs = []
        for _ in range(int(g.integers(0, 20))):
            if g.random() < 0.5:
                decs.append(OS.DecodeQoS(True, float(g.uniform(0, 100)), slo_ttft=6.0, slo_tbt=0.05,
                                         next_token=int(g.integers(1, 500))))
            else:
                decs.append(OS.DecodeQoS(False, float(g.uniform(0, 100)), slo_ttlt=float(g.choice([600, 1800])),
                                         est_remaining=int(g.integers(0, 900))))
        now = float(g.uniform(0, 200))
        assert ny.min_slack(decs, now) == pytest.approx(OS.min_slack(decs, now), rel=1e-15, abs=1e-15)


def test_iteration_predictor_closed_form_and_committed_fit():
    """Full-iteration mode (niyama_predictor_set_iteration): t = c0 + c1 T + lin(T) + layers * t_attn with
    lin piecewise linear (hand-computed), and profiles/iteration_fit.json reproduces through the C ABI
    (the paper's predictor scope): held-out p95 <= 5 %, max <= 7 % (final kernel: 4.2 % / 6.3 %;
    4.4 % / 5.3 % and 3.8 % / 4.8 % on earlier round-2 kernels)."""
    pr = ny.Predictor.from_params(CFG, THETA)
    d = W.BatchDesc([0], [1536], [512], list(range(1, 65)), [2048] * 64)
    a = pr.predict(d)
    pr.set_iteration(32, [16, 1024, 4096], [0.002, 0.010, 0.040], c0=1e-4, c1=2e-7)
    T = 576
    lin = 0.002 + (0.010 - 0.002) * (T - 16) / (1024 - 16)
    assert pr.predict(d) == pytest.approx(1e-4 + 2e-7 * T + lin + 32 * a, rel=1e-12)
    big = W.BatchDesc([0], [0], [2048], list(range(1, 2150)), [5] * 2149)   # T = 4197 > 4096: extrapolated
    assert pr.predict(big) > 0
    with pytest.raises(ny.NiyamaError):
        pr.set_iteration(32, [16, 16], [0.1, 0.2])              # tokens must ascend
    pr.set_iteration(0)
    assert pr.predict(d) == a
    fj = json.load(open(os.path.join(ROOT, "profiles", "iteration_fit.json")))
    sw = json.load(open(os.path.join(ROOT, fj["sweep"])))
    pf = json.load(open(os.path.join(ROOT, "profiles", "predictor_fit.json")))
    p2 = ny.Predictor.from_params(CFG, pf["theta"])
    lin = sorted(sw["linear"], key=lambda x: x["T"])
    p2.set_iteration(sw["layers"], [x["T"] for x in lin], [x["seconds"] for x in lin])

    def desc(r):
        c = r["chunk"]
        return W.BatchDesc([0] if c else [], [r["offset"]] if c else [], [c] if c else [], list(range(1, r["D"] + 1)),
                           list(r["ctx"]))
    train = [r for r in sw["points"] if (r["kind"] == "grid" and r["seed"] != 2) or r["kind"] == "random"]
    held = [r for r in sw["points"] if r["kind"] == "offgrid" or (r["kind"] == "grid" and r["seed"] == 2)]
    p2.fit_iteration([desc(r) for r in train], [r["seconds"] for r in train])
    err = np.abs([p2.predict(desc(r)) / r["seconds"] - 1 for r in held])
    assert float(err.max()) == pytest.approx(fj["errors"]["analytic"]["heldout"]["max"], rel=1e-9)
    assert float(np.percentile(err, 95)) <= 0.05 and float(err.max()) <= 0.07 and len(held) >= 30


def test_gather_window_host_validation():
    """§8(f)2 entry points validate before touching a device: no device -> EUNSUPPORTED;
    the one-process group checks rank/world/shape consistency (EINVAL)."""
    import paper_2503_22562_b200 as ny
    kv = ny.KVCache(1, 8, 2, 128, 16, dtype="bf16", device=None)
    with pytest.raises(ny.NiyamaError) as e:
        kv.gather_window(16)
    assert e.value.status == 7
    ranks = [ny.KVCache(1, 8, 2, 128, 16, dtype="bf16", world_size=2, rank=r, device=None) for r in range(2)]
    with pytest.raises(ny.NiyamaError) as e:
        ny.debug_gather_group(ranks, 16)
    assert e.value.status == 7
    with pytest.raises(ny.NiyamaError) as e:
        ny.debug_gather_group(ranks[::-1], 16)     # kvs[r] must be rank r (checked after the device check)
    assert e.value.status in (1, 7)
    with pytest.raises(ny.NiyamaError) as e:
        ny.debug_gather_group([], 16)
    assert e.value.status == 1


def test_committed_l70b_fit_reproduces():
    """profiles/predictor_fit_l70b.json (config-4 head shapes, Hq 64 / Hkv 8, the launch at g = 8
    with CTA pairs and producer-warp decode): the recorded predictions reproduce through the C ABI
    and the held-out errors are the file's own (final sweep: p50 1.1 %, p95 5.5 %, max 16.6 %, the
    worst at chunk 256 with few decodes as at L8B; an earlier sweep of the previous kernel: max 7.1 %)."""
    fj = json.load(open(os.path.join(ROOT, "profiles", "predictor_fit_l70b.json")))
    sw = json.load(open(os.path.join(ROOT, fj["sweep"])))
    assert sw["config"] == "l70b"
    pr = ny.Predictor.from_params(ny.Predictor.shape_cfg(64, 8, 128, "bf16"), fj["theta"])
    byk = {(p["kind"], p["seed"], p["chunk"], p["D"]): p for p in fj["points"]}
    held = []
    for r in sw["points"]:
        c = r["chunk"]
        d = W.BatchDesc([0] if c else [], [r["offset"]] if c else [], [c] if c else [], list(range(1, r["D"] + 1)),
                        list(r["ctx"]))
        rec = byk[(r["kind"], r["seed"], r["chunk"], r["D"])]
        assert pr.predict(d) == pytest.approx(rec["predicted"], rel=1e-12)
        if r["kind"] == "offgrid" or (r["kind"] == "grid" and r["seed"] == 2):
            held.append(pr.predict(d) / r["seconds"] - 1)
    held = np.abs(held)
    assert len(held) == fj["fit"]["heldout_points"] == 60
    assert float(held.max()) == pytest.approx(fj["heldout_rel_err"]["max"], rel=1e-9)
    assert float(np.median(held)) <= 0.02 and float(np.percentile(held, 95)) <= 0.06 and float(held.max()) <= 0.2

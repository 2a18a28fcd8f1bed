"""Test-side glue: run a workload through the C-ABI library on cuda:0 and through
the fp64 oracle on the same seeded inputs (tests only — imports both sides)."""
from __future__ import annotations

import math

import numpy as np
import torch

import workloads as W
from oracle import attention as OA
from oracle.kvcache import KVPool

TOL_MAX_ABS = 2e-2   # north_star: bf16-in / fp32-accumulate attention
TOL_REL_L2 = 5e-3


def to_dev(x: np.ndarray, dtype: str) -> torch.Tensor:
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def to_host_f64(t: torch.Tensor, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return OA.to_f64(t.view(torch.int16).cpu().numpy().view(np.uint16), "bf16")
    return t.double().cpu().numpy()


def stored_bits(t: torch.Tensor, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


class Run:
    """Executes every step of a workload through libniyama (append every step,
    attention on the final step)."""

    def __init__(self, wl: W.Workload, layers: int = 1, extra_blocks: int = 0, kv=None, scale: float = 0.0,
                 fused: bool = False, tuning=None):
        """fused: the final step's append runs inside the attention launch
        (niyama_append_attention) instead of its own launch."""
        import paper_2503_22562_b200 as ny
        s = wl.shape
        self.wl, self.s, self.fused = wl, s, fused
        self.kv = kv or ny.KVCache(layers, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + extra_blocks,
                                   block_size=s.block_size, dtype=s.dtype, device=0)
        if tuning:
            self.kv.set_tuning(**tuning)
        self.plans = []
        for n, st in enumerate(wl.steps):
            p = self.kv.plan(st.desc)
            self.plans.append(p)
            if fused and n == len(wl.steps) - 1:
                continue
            for layer in range(layers):
                self.kv.append(p, layer, to_dev(st.k, s.dtype), to_dev(st.v, s.dtype))
        self.plan = self.plans[-1]
        self.scale = scale

    def attention(self, layer: int = 0, q: np.ndarray | None = None):
        s, st = self.s, self.wl.final
        q = st.q if q is None else q
        T = st.desc.num_rows
        qd = to_dev(q, s.dtype)
        tdt = torch.bfloat16 if s.dtype == "bf16" else torch.float32
        o = torch.full((s.num_q_heads, T, s.head_dim), float("nan"), dtype=tdt, device="cuda")
        lse = torch.full((s.num_q_heads, T), float("nan"), dtype=torch.float32, device="cuda")
        if self.fused:
            self.kv.append_attention(self.plan, layer, to_dev(st.k, s.dtype), to_dev(st.v, s.dtype), qd, o, lse,
                                     self.scale)
        else:
            self.kv.attention(self.plan, layer, qd, o, lse, self.scale)
        torch.cuda.synchronize()
        return o, lse


def oracle_for(wl: W.Workload, rows=None, scale=None):
    s = wl.shape
    pool = KVPool(1, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
    plan = None
    for st in wl.steps:
        plan = pool.plan(st.desc)
        pool.append(0, plan, st.k, st.v)
    O, L = OA.hybrid_attention(pool, 0, plan, wl.final.q, s.num_q_heads, scale=scale, rows=rows)
    return pool, plan, O, L


def errors(o_gpu: np.ndarray, o_ref: np.ndarray):
    m = ~np.isnan(o_ref)
    diff = o_gpu[m] - o_ref[m]
    max_abs = float(np.abs(diff).max()) if diff.size else 0.0
    rel = float(np.linalg.norm(diff) / max(np.linalg.norm(o_ref[m]), 1e-30)) if diff.size else 0.0
    return max_abs, rel


def assert_close(o_gpu, o_ref, lse_gpu=None, lse_ref=None, max_abs=TOL_MAX_ABS, rel_l2=TOL_REL_L2, lse_tol=1e-3):
    ma, rl = errors(o_gpu, o_ref)
    assert np.isfinite(o_gpu[~np.isnan(o_ref)]).all(), "non-finite outputs"
    assert ma <= max_abs and rl <= rel_l2, f"max_abs={ma:.3e} rel_l2={rl:.3e}"
    if lse_gpu is not None:
        m = ~np.isnan(lse_ref)
        d = float(np.abs(lse_gpu[m] - lse_ref[m]).max()) if m.any() else 0.0
        assert d <= lse_tol, f"|dLSE|={d:.3e}"
    return ma, rl

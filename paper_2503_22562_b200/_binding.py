"""ctypes binding of libniyama.so (include/niyama.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels; there is no CPU
fallback, and importing this module fails loudly when the library is missing."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libniyama.so")

OK, EINVAL, ENOBLOCKS, ENOSEQ, ESTATE, ECUDA, ENCCL, EUNSUPPORTED = range(8)
STATUS_NAMES = ["OK", "EINVAL", "ENOBLOCKS", "ENOSEQ", "ESTATE", "ECUDA", "ENCCL", "EUNSUPPORTED"]
BF16, F32 = 0, 1
DEVICE_NONE = -1
NUM_PARAMS = 16
# the config-3 fit of round 2 (L8B shapes, profiles/predictor_fit.json; tools/fit_predictor.py)
DEFAULT_THETA = (1.8615542699363073e-05, 4.3100249351440104e-11, 0.0, 0.0, 1.823173461287965e-09, 1.0,
                 9.032153394238483e-07, 3.309503023249454e-08, 1.6819914137084094e-07, 7.7212032074647,
                 43416718287.28031, 2.1810731598188094e-08, 7443378861402.669,
                 0.22390466300385214, 84583517506.78802, 0.0010000000000000002)
PARAM_NAMES = ["c0 (s)", "per row c+D (s)", "per decode (s)", "per ctx token (s)", "per unit (s)", "kappa (T_sim)",
               "tau0 (s/step)", "tau_p (s/step)", "tau_d (s/step)", "sigma (steps/tile)", "r_w (B/s per warp)",
               "u0 (s/unit)", "BW (B/s)", "gamma", "r_cta (B/s)", "sigma0 (steps/CTA)"]


class NiyamaError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {message}")
        self.status = status
        self.code = status


class KVConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("block_size", C.c_int32), ("num_blocks", C.c_int32),
                ("dtype", C.c_int), ("world_size", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32)]


class BatchDescC(C.Structure):
    _fields_ = [("num_prefill", C.c_int32), ("prefill_seq", C.POINTER(C.c_int64)),
                ("prefill_offset", C.POINTER(C.c_int32)), ("prefill_len", C.POINTER(C.c_int32)),
                ("num_decode", C.c_int32), ("decode_seq", C.POINTER(C.c_int64)),
                ("decode_ctx", C.POINTER(C.c_int32)), ("tier", C.POINTER(C.c_uint8))]


class PlanInfo(C.Structure):
    _fields_ = [("num_rows", C.c_int32), ("num_prefill_rows", C.c_int32), ("num_decode", C.c_int32),
                ("num_prefill_tiles", C.c_int32), ("num_decode_units", C.c_int32), ("split_len", C.c_int32),
                ("rows_per_tile", C.c_int32), ("prefill_ctas", C.c_int32), ("sum_ctx", C.c_int64)]


class Tuning(C.Structure):
    _fields_ = [("prefill_ctas", C.c_int32), ("split_len", C.c_int32), ("tail_div", C.c_int32),
                ("tail_min", C.c_int32), ("grid_cap", C.c_int32), ("plan_copy_stream", C.c_int32),
                ("decode_path", C.c_int32), ("prefill_split", C.c_int32), ("prefill_pairs", C.c_int32)]


class SampleC(C.Structure):
    _fields_ = [("chunk_len", C.c_int32), ("chunk_offset", C.c_int32), ("num_decode", C.c_int32),
                ("sum_ctx", C.c_int64), ("seconds", C.c_double)]


class FitOptionsC(C.Structure):
    _fields_ = [("start", C.POINTER(C.c_double)), ("max_evals", C.c_int32), ("subsample", C.c_int32)]


class PredictInfoC(C.Structure):
    _fields_ = [("grid", C.c_int32), ("prefill_ctas", C.c_int32), ("split_len", C.c_int32),
                ("small_piece", C.c_int32), ("warps_per_cta", C.c_int32), ("prefill_parts_target", C.c_int32),
                ("num_units", C.c_int64), ("sim_seconds", C.c_double), ("seconds", C.c_double)]


class DecodeQoSC(C.Structure):
    _fields_ = [("interactive", C.c_int32), ("next_token", C.c_int32), ("est_remaining", C.c_int32),
                ("reserved", C.c_int32), ("t_arrival", C.c_double), ("slo_ttft", C.c_double),
                ("slo_tbt", C.c_double), ("slo_ttlt", C.c_double)]


class SchedConfigC(C.Structure):
    _fields_ = [("policy", C.c_int32), ("preemption", C.c_int32), ("dynamic_chunk", C.c_int32),
                ("fixed_chunk", C.c_int32), ("max_chunk", C.c_int32), ("relegation", C.c_int32),
                ("multi_fill", C.c_int32), ("history_min_samples", C.c_int32), ("alpha", C.c_double),
                ("prior_mean", C.c_double), ("prior_std", C.c_double), ("decode_token_s", C.c_double),
                ("layers", C.c_double), ("fixed_s", C.c_double), ("kv_token_budget", C.c_int64)]


class QoSSpecC(C.Structure):
    _fields_ = [("interactive", C.c_int32), ("reserved", C.c_int32), ("slo_ttft", C.c_double),
                ("slo_tbt", C.c_double), ("slo_ttlt", C.c_double)]


class SchedBatchC(C.Structure):
    _fields_ = [("desc", BatchDescC), ("chunk_budget", C.c_int32), ("infeasible", C.c_int32),
                ("predicted_s", C.c_double), ("min_slack_s", C.c_double), ("num_relegated", C.c_int32),
                ("relegated", C.POINTER(C.c_int64))]


class RequestInfoC(C.Structure):
    _fields_ = [("state", C.c_int32), ("relegated", C.c_int32), ("prefill_done", C.c_int32),
                ("decoded", C.c_int32), ("prompt", C.c_int32), ("low", C.c_int32)]


def _load():
    # NIYAMA_LIB_PATH: load an alternate build of the same library (A/B experiments
    # with tools/build_variant.py); the default is the in-tree libniyama.so.
    path = os.environ.get("NIYAMA_LIB_PATH", LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built: run `python paper_2503_22562_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    vp, i32, i64, st = C.c_void_p, C.c_int32, C.c_int64, C.c_int
    sigs = {
        "niyama_last_error": ([], C.c_char_p),
        "niyama_version": ([], C.c_char_p),
        "niyama_kv_create": ([C.POINTER(KVConfig), C.POINTER(vp)], st),
        "niyama_kv_destroy": ([vp], None),
        "niyama_kv_release": ([vp, i64], st),
        "niyama_kv_truncate": ([vp, i64, i32], st),
        "niyama_kv_block_table": ([vp, i64, C.POINTER(i32), i32, C.POINTER(i32)], st),
        "niyama_kv_seq_len": ([vp, i64, C.POINTER(i32)], st),
        "niyama_kv_num_free": ([vp, C.POINTER(i32)], st),
        "niyama_kv_gather": ([vp, i32, i64, i32, vp, vp, vp], st),
        "niyama_plan_create": ([vp, C.POINTER(BatchDescC), vp, C.POINTER(vp)], st),
        "niyama_plan_destroy": ([vp], None),
        "niyama_plan_get_info": ([vp, C.POINTER(PlanInfo)], st),
        "niyama_plan_rollback": ([vp, vp], st),
        "niyama_plan_slots": ([vp, C.POINTER(i32), C.POINTER(i32), i32], st),
        "niyama_kv_append": ([vp, vp, i32, vp, vp, vp], st),
        "niyama_hybrid_attention": ([vp, vp, i32, vp, vp, vp, C.c_float, vp], st),
        "niyama_append_attention": ([vp, vp, i32, vp, vp, vp, vp, vp, C.c_float, vp], st),
        "niyama_debug_trace": ([vp, vp], st),
        "niyama_kv_get_tuning": ([vp, C.POINTER(Tuning)], st),
        "niyama_kv_set_tuning": ([vp, C.POINTER(Tuning)], st),
        "niyama_predictor_bind": ([vp, vp], st),
        "niyama_comm_init": ([vp, vp], st),
        "niyama_get_unique_id": ([vp], st),
        "niyama_allgather_heads": ([vp, vp, vp, vp, vp], st),
        "niyama_gather_create": ([vp, i32, C.POINTER(vp)], st),
        "niyama_gather_destroy": ([vp], st),
        "niyama_debug_gather_group": ([C.POINTER(vp), i32, i32, C.POINTER(vp)], st),
        "niyama_attention_gather": ([vp, vp, i32, vp, vp, vp, vp, C.c_float, C.POINTER(vp), C.POINTER(vp), vp], st),
        "niyama_predictor_fit": ([C.POINTER(KVConfig), C.POINTER(SampleC), i32, C.POINTER(vp)], st),
        "niyama_predictor_fit_batches": ([C.POINTER(KVConfig), C.POINTER(BatchDescC), C.POINTER(C.c_double), i32,
                                          C.POINTER(FitOptionsC), C.POINTER(vp)], st),
        "niyama_predict_detail": ([vp, C.POINTER(BatchDescC), C.POINTER(PredictInfoC)], st),
        "niyama_predictor_set_iteration": ([vp, i32, C.POINTER(i32), C.POINTER(C.c_double), i32, C.c_double,
                                            C.c_double], st),
        "niyama_predictor_fit_iteration": ([vp, C.POINTER(BatchDescC), C.POINTER(C.c_double), i32], st),
        "niyama_predictor_from_params": ([C.POINTER(KVConfig), C.POINTER(C.c_double), C.POINTER(vp)], st),
        "niyama_predictor_params": ([vp, C.POINTER(C.c_double)], st),
        "niyama_predict_iter_time": ([vp, C.POINTER(BatchDescC)], C.c_double),
        "niyama_max_feasible_chunk": ([vp, C.POINTER(BatchDescC), i32, i32, C.c_double, i32, C.POINTER(i32),
                                       C.POINTER(i32)], st),
        "niyama_predictor_destroy": ([vp], None),
        "niyama_min_slack": ([C.POINTER(DecodeQoSC), i32, C.c_double, C.POINTER(C.c_double)], st),
        "niyama_sched_config_default": ([C.POINTER(SchedConfigC)], None),
        "niyama_sched_create": ([C.POINTER(SchedConfigC), vp, C.POINTER(vp)], st),
        "niyama_sched_destroy": ([vp], None),
        "niyama_sched_submit": ([vp, i64, C.c_double, i32, C.POINTER(QoSSpecC), i32, i32, i32], st),
        "niyama_sched_next_batch": ([vp, C.c_double, C.POINTER(SchedBatchC)], st),
        "niyama_sched_complete": ([vp, C.c_double, C.POINTER(i64), i32], st),
        "niyama_sched_request": ([vp, i64, C.POINTER(RequestInfoC)], st),
        "niyama_sched_counts": ([vp, C.POINTER(i32)], st),
        "niyama_sched_priority": ([vp, i64, C.c_double, C.POINTER(C.c_double), C.POINTER(i32)], st),
    }
    for name, (args, res) in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def _check(status: int):
    if status != OK:
        raise NiyamaError(status, lib.niyama_last_error().decode())


def _ptr(x) -> Optional[int]:
    """Device/host pointer of a torch tensor (must be contiguous) or a raw int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if hasattr(x, "is_contiguous") and not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(f"expected a tensor or an int pointer, got {type(x)}")


def _stream(s) -> Optional[int]:
    if s is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover - torch is part of the image
            pass
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


class _Desc:
    """Keeps the numpy buffers of a batch descriptor alive while the C struct is used."""

    def __init__(self, desc):
        ps = getattr(desc, "prefill_seq", []) or []
        ds = getattr(desc, "decode_seq", []) or []
        self.ps = np.ascontiguousarray(ps, dtype=np.int64)
        self.po = np.ascontiguousarray(getattr(desc, "prefill_offset", []) or [], dtype=np.int32)
        self.pl = np.ascontiguousarray(getattr(desc, "prefill_len", []) or [], dtype=np.int32)
        self.ds = np.ascontiguousarray(ds, dtype=np.int64)
        self.dc = np.ascontiguousarray(getattr(desc, "decode_ctx", []) or [], dtype=np.int32)
        tier = getattr(desc, "tier", None)
        self.tier = None if tier is None else np.ascontiguousarray(tier, dtype=np.uint8)
        if len(self.po) != len(self.ps) or len(self.pl) != len(self.ps) or len(self.dc) != len(self.ds):
            raise ValueError("descriptor arrays disagree in length")
        if self.tier is not None and len(self.tier) != len(self.ps) + len(self.ds):
            raise ValueError("tier array length")

        def p(a, t):
            return a.ctypes.data_as(C.POINTER(t)) if a is not None and len(a) else None

        self.c = BatchDescC(len(self.ps), p(self.ps, C.c_int64), p(self.po, C.c_int32), p(self.pl, C.c_int32),
                            len(self.ds), p(self.ds, C.c_int64), p(self.dc, C.c_int32), p(self.tier, C.c_uint8))


def _cfg(num_layers, num_q_heads, num_kv_heads, head_dim, block_size, num_blocks, dtype, world_size, rank, device):
    dt = {"bf16": BF16, "f32": F32, BF16: BF16, F32: F32}[dtype]
    return KVConfig(num_layers, num_q_heads, num_kv_heads, head_dim, block_size, num_blocks, dt, world_size, rank,
                    DEVICE_NONE if device is None else device)


class Plan:
    def __init__(self, kv: "KVCache", handle: int):
        self.kv = kv
        self.handle = handle

    def info(self) -> PlanInfo:
        out = PlanInfo()
        _check(lib.niyama_plan_get_info(self.handle, C.byref(out)))
        return out

    def slots(self):
        n = self.info().num_rows
        blk = np.zeros(max(n, 1), np.int32)
        slot = np.zeros(max(n, 1), np.int32)
        _check(lib.niyama_plan_slots(self.handle, blk.ctypes.data_as(C.POINTER(C.c_int32)),
                                     slot.ctypes.data_as(C.POINTER(C.c_int32)), n))
        return list(zip(blk[:n].tolist(), slot[:n].tolist()))

    def rollback(self):
        _check(lib.niyama_plan_rollback(self.kv.handle, self.handle))

    def close(self):
        if self.handle:
            lib.niyama_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class KVCache:
    """Library-owned paged KV pool (niyama_kv)."""

    def __init__(self, num_layers: int, num_q_heads: int, num_kv_heads: int, head_dim: int, num_blocks: int,
                 block_size: int = 16, dtype: str = "bf16", world_size: int = 1, rank: int = 0,
                 device: Optional[int] = 0):
        self.cfg = _cfg(num_layers, num_q_heads, num_kv_heads, head_dim, block_size, num_blocks, dtype, world_size,
                        rank, device)
        h = C.c_void_p()
        _check(lib.niyama_kv_create(C.byref(self.cfg), C.byref(h)))
        self.handle = h.value
        self.dtype = dtype

    # -- bookkeeping
    def plan(self, desc, stream=None) -> Plan:
        d = desc if isinstance(desc, _Desc) else _Desc(desc)
        h = C.c_void_p()
        _check(lib.niyama_plan_create(self.handle, C.byref(d.c), _stream(stream), C.byref(h)))
        plan = Plan(self, h.value)
        if not hasattr(self, "_plans"):
            import weakref
            self._plans = weakref.WeakSet()
        self._plans.add(plan)
        return plan

    def release(self, seq: int):
        _check(lib.niyama_kv_release(self.handle, int(seq)))

    def truncate(self, seq: int, new_len: int):
        _check(lib.niyama_kv_truncate(self.handle, int(seq), int(new_len)))

    def block_table(self, seq: int):
        n = C.c_int32()
        _check(lib.niyama_kv_block_table(self.handle, int(seq), None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int32)
        _check(lib.niyama_kv_block_table(self.handle, int(seq), out.ctypes.data_as(C.POINTER(C.c_int32)), n.value,
                                         C.byref(n)))
        return out[: n.value].tolist()

    def seq_len(self, seq: int) -> int:
        n = C.c_int32()
        _check(lib.niyama_kv_seq_len(self.handle, int(seq), C.byref(n)))
        return n.value

    def num_free(self) -> int:
        n = C.c_int32()
        _check(lib.niyama_kv_num_free(self.handle, C.byref(n)))
        return n.value

    # -- device work
    def append(self, plan: Plan, layer: int, k_new, v_new, stream=None):
        _check(lib.niyama_kv_append(self.handle, plan.handle, layer, _ptr(k_new), _ptr(v_new), _stream(stream)))

    def attention(self, plan: Plan, layer: int, q, o, lse=None, scale: float = 0.0, stream=None):
        _check(lib.niyama_hybrid_attention(self.handle, plan.handle, layer, _ptr(q), _ptr(o), _ptr(lse),
                                           float(scale), _stream(stream)))

    def append_attention(self, plan: Plan, layer: int, k_new, v_new, q, o, lse=None, scale: float = 0.0,
                         stream=None):
        _check(lib.niyama_append_attention(self.handle, plan.handle, layer, _ptr(k_new), _ptr(v_new), _ptr(q),
                                           _ptr(o), _ptr(lse), float(scale), _stream(stream)))

    def gather(self, layer: int, seq: int, n: int, k_out, v_out, stream=None):
        _check(lib.niyama_kv_gather(self.handle, layer, int(seq), n, _ptr(k_out), _ptr(v_out), _stream(stream)))

    def debug_trace(self, buf):
        _check(lib.niyama_debug_trace(self.handle, _ptr(buf)))

    def tuning(self) -> Tuning:
        t = Tuning()
        _check(lib.niyama_kv_get_tuning(self.handle, C.byref(t)))
        return t

    def set_tuning(self, **fields):
        """Change named niyama_tuning fields (include/niyama.h); the others keep their values."""
        t = self.tuning()
        for k, v in fields.items():
            if not hasattr(t, k):
                raise AttributeError(f"niyama_tuning has no field {k}")
            setattr(t, k, int(v))
        _check(lib.niyama_kv_set_tuning(self.handle, C.byref(t)))

    def comm_init(self, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib.niyama_comm_init(self.handle, buf))

    def allgather_heads(self, plan: Plan, o_full, lse_full=None, stream=None):
        _check(lib.niyama_allgather_heads(self.handle, plan.handle, _ptr(o_full), _ptr(lse_full), _stream(stream)))

    def gather_window(self, max_rows: int) -> "GatherWindow":
        """§8(f)2: the symmetric output window of the fused all-gather (collective: every rank)."""
        h = C.c_void_p()
        _check(lib.niyama_gather_create(self.handle, int(max_rows), C.byref(h)))
        w = GatherWindow(self, h.value)
        if not hasattr(self, "_windows"):
            import weakref
            self._windows = weakref.WeakSet()
        self._windows.add(w)
        return w

    def attention_gather(self, plan: Plan, layer: int, q, window: "GatherWindow", k_new=None, v_new=None,
                         scale: float = 0.0, stream=None):
        """Append (optional) + attention + head all-gather in ONE launch (niyama_attention_gather).
        Returns torch views (o_full [Hq_all][T][d] bf16, lse_full [Hq_all][T] f32) of the window
        buffer the launch fills; valid until the call after next."""
        o = C.c_void_p()
        lse = C.c_void_p()
        _check(lib.niyama_attention_gather(self.handle, plan.handle, layer, _ptr(k_new), _ptr(v_new), _ptr(q),
                                           window.handle, float(scale), C.byref(o), C.byref(lse), _stream(stream)))
        T = plan.info().num_rows
        hq = self.cfg.num_q_heads   # global head count (every rank's heads are in the window)
        return (_device_view(o.value, (hq, T, self.cfg.head_dim), "<V2", self.cfg.device),
                _device_view(lse.value, (hq, T), "<f4", self.cfg.device))

    def close(self):
        if getattr(self, "handle", None):
            # a plan's buffers come from this cache's memory pool: destroy live plans first;
            # gather windows use the communicator the cache owns
            for plan in list(getattr(self, "_plans", ())):
                plan.close()
            for w in list(getattr(self, "_windows", ())):
                w.close()
            lib.niyama_kv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GatherWindow:
    """niyama_gather: NCCL symmetric window holding the fused all-gather's outputs."""

    def __init__(self, kv: KVCache, handle: int):
        self.kv = kv
        self.handle = handle

    def close(self):
        if self.handle:
            h, self.handle = self.handle, None
            _check(lib.niyama_gather_destroy(h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def debug_gather_group(kvs, max_rows: int):
    """niyama_debug_gather_group: windows of n one-device ranks (kvs[r] = rank r of world n)
    cross-linked as peers (tests of the multi-rank protocol on one GPU)."""
    n = len(kvs)
    hs = (C.c_void_p * n)(*[kv.handle for kv in kvs])
    outs = (C.c_void_p * n)()
    _check(lib.niyama_debug_gather_group(hs, n, int(max_rows), outs))
    ws = [GatherWindow(kv, outs[r]) for r, kv in enumerate(kvs)]
    for kv, w in zip(kvs, ws):
        if not hasattr(kv, "_windows"):
            import weakref
            kv._windows = weakref.WeakSet()
        kv._windows.add(w)
    return ws


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _device_view(ptr, shape, typestr, device):
    """A torch tensor aliasing library-owned device memory (no copy)."""
    import torch
    if typestr == "<V2":  # bf16: viewed through int16 (no bf16 typestr in the interface)
        return torch.as_tensor(_CudaArray(ptr, shape, "<i2"), device=f"cuda:{device}").view(torch.bfloat16)
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=f"cuda:{device}")


def get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.niyama_get_unique_id(buf))
    return buf.raw


class Predictor:
    """Iteration-time predictor (niyama_predictor): the a8 event model of include/niyama.h.

    Parameters (PARAM_NAMES): theta[0:6] linear weights of [1, c+D, D, sum ctx, units, T_sim];
    theta[6:13] the event model's tau0, tau_p, tau_d, sigma, r_w, u0, BW."""

    def __init__(self, handle: int):
        self.handle = handle

    @staticmethod
    def shape_cfg(num_q_heads, num_kv_heads, head_dim, dtype="bf16", world_size=1):
        return _cfg(1, num_q_heads, num_kv_heads, head_dim, 16, 1, dtype, world_size, 0, None)

    @classmethod
    def fit(cls, cfg: KVConfig, samples: Sequence) -> "Predictor":
        """Summary samples (chunk_len, chunk_offset, num_decode, sum_ctx, seconds)."""
        arr = (SampleC * len(samples))(*[SampleC(s.chunk_len, s.chunk_offset, s.num_decode, s.sum_ctx, s.seconds)
                                         for s in samples])
        h = C.c_void_p()
        _check(lib.niyama_predictor_fit(C.byref(cfg), arr, len(samples), C.byref(h)))
        return cls(h.value)

    @classmethod
    def fit_batches(cls, cfg: KVConfig, batches: Sequence, seconds: Sequence[float], start=None, max_evals=0,
                    subsample=0) -> "Predictor":
        """Measured launches: batches (descriptor objects or `Batch`) and their seconds."""
        ds = [b if isinstance(b, _Desc) else _Desc(b) for b in batches]
        arr = (BatchDescC * len(ds))(*[d.c for d in ds])
        sec = (C.c_double * len(ds))(*[float(x) for x in seconds])
        opt = FitOptionsC(None, int(max_evals), int(subsample))
        if start is not None:
            st = (C.c_double * NUM_PARAMS)(*[float(x) for x in start])
            opt.start = st
        h = C.c_void_p()
        _check(lib.niyama_predictor_fit_batches(C.byref(cfg), arr, sec, len(ds), C.byref(opt), C.byref(h)))
        return cls(h.value)

    def set_iteration(self, layers: int, tokens=(), seconds=(), c0: float = 0.0, c1: float = 0.0) -> "Predictor":
        """Full-iteration mode (niyama_predictor_set_iteration); layers = 0 switches it off."""
        n = len(tokens)
        tk = (C.c_int32 * max(1, n))(*[int(x) for x in tokens])
        sc = (C.c_double * max(1, n))(*[float(x) for x in seconds])
        _check(lib.niyama_predictor_set_iteration(self.handle, int(layers), tk, sc, n, float(c0), float(c1)))
        return self

    def fit_iteration(self, batches, seconds) -> "Predictor":
        ds = [b if isinstance(b, _Desc) else _Desc(b) for b in batches]
        arr = (BatchDescC * len(ds))(*[d.c for d in ds])
        sec = (C.c_double * len(ds))(*[float(x) for x in seconds])
        _check(lib.niyama_predictor_fit_iteration(self.handle, arr, sec, len(ds)))
        return self

    def detail(self, desc) -> dict:
        d = desc if isinstance(desc, _Desc) else _Desc(desc)
        out = PredictInfoC()
        _check(lib.niyama_predict_detail(self.handle, C.byref(d.c), C.byref(out)))
        return dict(grid=out.grid, prefill_ctas=out.prefill_ctas, split_len=out.split_len,
                    small_piece=out.small_piece, warps_per_cta=out.warps_per_cta,
                    parts_target=out.prefill_parts_target, units=out.num_units,
                    sim=out.sim_seconds, seconds=out.seconds)

    @classmethod
    def from_params(cls, cfg: KVConfig, theta) -> "Predictor":
        if len(theta) != NUM_PARAMS:
            raise ValueError(f"theta needs {NUM_PARAMS} values")
        th = (C.c_double * NUM_PARAMS)(*[float(x) for x in theta])
        h = C.c_void_p()
        _check(lib.niyama_predictor_from_params(C.byref(cfg), th, C.byref(h)))
        return cls(h.value)

    def bind(self, kv: "KVCache") -> "Predictor":
        """Model kv's launches: its SM count and tuning (niyama_predictor_bind)."""
        _check(lib.niyama_predictor_bind(self.handle, kv.handle))
        return self

    def params(self) -> np.ndarray:
        th = (C.c_double * NUM_PARAMS)()
        _check(lib.niyama_predictor_params(self.handle, th))
        return np.array(list(th))

    def predict(self, desc) -> float:
        d = desc if isinstance(desc, _Desc) else _Desc(desc)
        return lib.niyama_predict_iter_time(self.handle, C.byref(d.c))

    def max_feasible_chunk(self, decode_ctx, chunk_offset, prefill_remaining, slack, max_chunk):
        """decode_ctx: a list of contexts or a prebuilt `Batch` holding the decodes."""
        if isinstance(decode_ctx, _Desc):
            d = decode_ctx
        else:
            class _D:
                pass
            dd = _D()
            dd.decode_seq = list(range(len(decode_ctx)))
            dd.decode_ctx = list(decode_ctx)
            d = _Desc(dd)
        c, inf = C.c_int32(), C.c_int32()
        _check(lib.niyama_max_feasible_chunk(self.handle, C.byref(d.c), chunk_offset, prefill_remaining,
                                             float(slack), max_chunk, C.byref(c), C.byref(inf)))
        return c.value, bool(inf.value)

    def __del__(self):
        try:
            if self.handle:
                lib.niyama_predictor_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


Batch = _Desc  # a batch descriptor marshalled once and reusable across calls


class DecodeQoS:
    """Python-side record of one running decode's QoS state (fields of `niyama_decode_qos`, include/niyama.h)."""

    __slots__ = ("interactive", "t_arrival", "slo_ttft", "slo_tbt", "slo_ttlt", "next_token", "est_remaining")

    def __init__(self, interactive, t_arrival, slo_ttft=0.0, slo_tbt=0.0, slo_ttlt=0.0, next_token=1,
                 est_remaining=1):
        self.interactive, self.t_arrival = bool(interactive), float(t_arrival)
        self.slo_ttft, self.slo_tbt, self.slo_ttlt = float(slo_ttft), float(slo_tbt), float(slo_ttlt)
        self.next_token, self.est_remaining = int(next_token), int(est_remaining)


class QoSArray:
    """niyama_decode_qos[] marshalled once (for per-iteration min_slack calls)."""

    def __init__(self, decodes):
        self.n = len(decodes)
        self.arr = (DecodeQoSC * max(1, self.n))(*[
            DecodeQoSC(int(bool(q.interactive)), int(q.next_token), int(q.est_remaining), 0, float(q.t_arrival),
                       float(q.slo_ttft), float(q.slo_tbt), float(q.slo_ttlt)) for q in decodes])

    def min_slack(self, now: float) -> float:
        out = C.c_double()
        _check(lib.niyama_min_slack(self.arr, self.n, float(now), C.byref(out)))
        return out.value


def min_slack(decodes, now: float) -> float:
    """decodes: objects with interactive, t_arrival, slo_ttft, slo_tbt, slo_ttlt, next_token, est_remaining."""
    arr = (DecodeQoSC * max(1, len(decodes)))(*[
        DecodeQoSC(int(bool(q.interactive)), int(q.next_token), int(q.est_remaining), 0, float(q.t_arrival),
                   float(q.slo_ttft), float(q.slo_tbt), float(q.slo_ttlt)) for q in decodes])
    out = C.c_double()
    _check(lib.niyama_min_slack(arr, len(decodes), float(now), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- §8(f)1 scheduler
POLICY = {"niyama": 0, "fcfs": 1, "edf": 2, "sjf": 3, "srpf": 4}
PREEMPT = {"never": 0, "selective": 1, "always": 2}
STATE_NAMES = ["prefill", "decode", "relegated", "done"]


class SchedBatch:
    """One iteration's batch from niyama_sched_next_batch (copied out of the scheduler's arrays)."""

    __slots__ = ("slices", "decodes", "tier", "budget", "infeasible", "predicted", "min_slack", "relegated", "raw")

    def __init__(self, c: SchedBatchC):
        d = c.desc
        self.slices = [(int(d.prefill_seq[i]), int(d.prefill_offset[i]), int(d.prefill_len[i]))
                       for i in range(d.num_prefill)]
        self.decodes = [(int(d.decode_seq[j]), int(d.decode_ctx[j])) for j in range(d.num_decode)]
        self.tier = [int(d.tier[i]) for i in range(d.num_prefill + d.num_decode)]
        self.budget, self.infeasible = int(c.chunk_budget), bool(c.infeasible)
        self.predicted, self.min_slack = float(c.predicted_s), float(c.min_slack_s)
        self.relegated = [int(c.relegated[i]) for i in range(c.num_relegated)]
        self.raw = c

    @property
    def empty(self) -> bool:
        return not self.slices and not self.decodes

    def desc(self):
        """A niyama_batch_desc for KVCache.plan (marshalled once)."""
        class _D:
            pass
        x = _D()
        x.prefill_seq = [s for s, _, _ in self.slices]
        x.prefill_offset = [o for _, o, _ in self.slices]
        x.prefill_len = [n for _, _, n in self.slices]
        x.decode_seq = [s for s, _ in self.decodes]
        x.decode_ctx = [c for _, c in self.decodes]
        x.tier = list(self.tier)
        return _Desc(x)


class Scheduler:
    """niyama_sched: the per-replica QoS scheduler core (include/niyama.h §8(f)1)."""

    def __init__(self, model: "Predictor", policy="niyama", preemption="selective", dynamic_chunk=True,
                 fixed_chunk=256, max_chunk=2048, relegation=True, multi_fill=True, history_min_samples=30,
                 alpha=0.0, prior_mean=415.0, prior_std=300.0, decode_token_s=0.05, layers=1.0, fixed_s=0.0,
                 kv_token_budget=0):
        cfg = SchedConfigC()
        lib.niyama_sched_config_default(C.byref(cfg))
        cfg.policy = POLICY[policy] if isinstance(policy, str) else int(policy)
        cfg.preemption = PREEMPT[preemption] if isinstance(preemption, str) else int(preemption)
        cfg.dynamic_chunk, cfg.fixed_chunk, cfg.max_chunk = int(bool(dynamic_chunk)), int(fixed_chunk), int(max_chunk)
        cfg.relegation, cfg.multi_fill = int(bool(relegation)), int(bool(multi_fill))
        cfg.history_min_samples = int(history_min_samples)
        cfg.alpha, cfg.prior_mean, cfg.prior_std = float(alpha), float(prior_mean), float(prior_std)
        cfg.decode_token_s = float(decode_token_s)
        cfg.layers, cfg.fixed_s = float(layers), float(fixed_s)
        cfg.kv_token_budget = int(kv_token_budget)
        self.model = model           # keep the borrowed predictor alive
        h = C.c_void_p()
        _check(lib.niyama_sched_create(C.byref(cfg), model.handle, C.byref(h)))
        self.handle = h.value

    def submit(self, rid, t_arrival, prompt, interactive, slo_ttft=0.0, slo_tbt=0.0, slo_ttlt=0.0, low=False,
               app=0, tier=0):
        q = QoSSpecC(int(bool(interactive)), 0, float(slo_ttft), float(slo_tbt), float(slo_ttlt))
        _check(lib.niyama_sched_submit(self.handle, int(rid), float(t_arrival), int(prompt), C.byref(q),
                                       int(bool(low)), int(app), int(tier)))

    def next_batch(self, now: float) -> SchedBatch:
        out = SchedBatchC()
        _check(lib.niyama_sched_next_batch(self.handle, float(now), C.byref(out)))
        return SchedBatch(out)

    def complete(self, now: float, finished: Sequence[int] = ()):
        arr = (C.c_int64 * max(1, len(finished)))(*[int(x) for x in finished])
        _check(lib.niyama_sched_complete(self.handle, float(now), arr, len(finished)))

    def request(self, rid) -> dict:
        out = RequestInfoC()
        _check(lib.niyama_sched_request(self.handle, int(rid), C.byref(out)))
        return dict(state=STATE_NAMES[out.state], relegated=bool(out.relegated), prefill_done=out.prefill_done,
                    decoded=out.decoded, prompt=out.prompt, low=bool(out.low))

    def counts(self) -> dict:
        arr = (C.c_int32 * 4)()
        _check(lib.niyama_sched_counts(self.handle, arr))
        return dict(zip(STATE_NAMES, list(arr)))

    def priority(self, rid, now: float):
        k, s = C.c_double(), C.c_int32()
        _check(lib.niyama_sched_priority(self.handle, int(rid), float(now), C.byref(k), C.byref(s)))
        return k.value, s.value

    def close(self):
        if self.handle:
            lib.niyama_sched_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

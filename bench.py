#!/usr/bin/env python
"""bench.py — hybrid-batch paged attention of Niyama (arXiv 2503.22562) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl niyama|reference] [--config l8b|l70b]

A STEP is one pass of the whole hot path over one
batch, i.e. one serving iteration: a1 min slack + max feasible chunk (host), a2
plan (host bookkeeping + one H2D, ONCE per iteration: the plan serves every
layer), then for each of the model's L attention layers (32 for Llama-3-8B,
--layers to change) a3 KV append (kernel) and a4-a6 the fused hybrid attention
launch (kernel) over that layer's own paged KV (+ a7 head all-gather, NCCL,
N>1), and a8 predictor eval (host).  The same batch is replayed every step
(sequences are truncated back after planning, host-only).  Default workload =
BASELINE config 2: Llama-3-8B attention shapes (32 q / 8 kv heads, d 128, bf16,
block 16), a 512-token prefill chunk at offset 1536 plus 64 decodes with ctx ~
U{1..4096} (PCG64 seed 0, sum ctx 133,674).  value = layer-tokens (T = 576 rows
x L layers) per second of device time, max over ranks (strong scaling: heads
are sharded over N GPUs, the batch is fixed).

Timing: CUDA events on the launching stream, W untimed warm-up steps, a
barrier + synchronize on both sides of exactly K timed steps.  L2: inputs
larger than L2 (556 MB of KV read per layer, every layer its own, vs 126 MB).  The
`roofline` object uses the attention launch's own per-launch event times.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hybrid-batch attn tokens/s & roofline % (Llama-3-8B shapes, chunk 512+64 dec)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="niyama", choices=["niyama", "reference"])
    ap.add_argument("--config", default="l8b", choices=["l8b", "l70b"])
    ap.add_argument("--layers", type=int, default=0,
                    help="attention layers per step (0 = the model's: 32 for Llama-3-8B, 80 for Llama-3-70B); one "
                         "plan serves all layers of the iteration (SURVEY 8(a) a2), each layer has its own KV")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--settle-s", type=float, default=1.0, help="untimed GPU work before warm-up (clock settle)")
    ap.add_argument("--host-only", action="store_true",
                    help="CPU check of the N-rank plumbing (gloo, NIYAMA_DEVICE_NONE pools): rank setup, replicated "
                         "planner, NCCL unique-id broadcast, a1/a2/a8 host steps; prints a line marked "
                         "impl=host-only (not a bench result)")
    ap.add_argument("--fused-append", action="store_true",
                    help="a3-a6 in one launch (niyama_append_attention) instead of niyama_kv_append + "
                         "niyama_hybrid_attention (measured slower on config 2: 113 vs 100 + 10 us)")
    ap.add_argument("--tuning", default="",
                    help="diagnostics: niyama_tuning fields for the timed KVCache, e.g. prefill_ctas=88,split_len=256 "
                         "(include/niyama.h; default = the planner's own choices)")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "fused"],
                    help="a7 head all-gather: nccl = niyama_allgather_heads after the launch (N > 1 only); fused = "
                         "niyama_attention_gather, the all-gather inside the attention launch (NVLink stores into "
                         "an NCCL symmetric window + flag barrier; run at every N, at N = 1 through the GPU's own "
                         "window mapping)")
    return ap.parse_args()


def workload(name):
    import workloads as W
    if name == "l8b":
        return W.config2_l8b()
    return W.config4_l70b()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def algorithmic(wl, hq, hkv):
    """B_KV = [sum(o+c) + sum ctx] * Hkv * d * 2 * elt; F = 4 d Hq [sum(c o + c(c+1)/2) + sum ctx]."""
    s, d = wl.shape, wl.final.desc
    tok = sum(o + c for o, c in zip(d.prefill_offset, d.prefill_len)) + sum(d.decode_ctx)
    pairs = sum(c * o + c * (c + 1) // 2 for o, c in zip(d.prefill_offset, d.prefill_len)) + sum(d.decode_ctx)
    B = tok * hkv * s.head_dim * 2 * s.elt_bytes
    F = 4.0 * s.head_dim * hq * pairs
    return B, F


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while running."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, line in self.lines:
            if not (t0 <= ts <= t1):
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N ranks on 127.0.0.1 (one process per GPU), forwarding
    its output; returns the exit code."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def dist_setup(n, host_only=False):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        gloo = host_only or os.environ.get("NIYAMA_BENCH_GLOO") is not None
        dist.init_process_group("gloo" if gloo else "nccl")
        pg = dist
    return rank, world, local, pg


def run_host_only(args, rank, world, dist):
    """--host-only: the N-rank plumbing of the real run on CPU (tests/test_bench_spawn.py).
    Every rank owns Hkv/N heads of a DEVICE_NONE pool, plans the config's batch with the
    replicated planner (no metadata exchange), receives the NCCL unique id broadcast by
    rank 0, and runs the a1/a2/a8 host steps; rank 0 checks every rank planned the same
    slots and prints one line."""
    import paper_2503_22562_b200 as ny
    wl = workload(args.config)
    s = wl.shape
    kv = ny.KVCache(1, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 64, block_size=s.block_size,
                    dtype=s.dtype, world_size=world, rank=rank, device=None)
    uid = [ny.get_unique_id() if rank == 0 else b""]
    if dist:
        dist.broadcast_object_list(uid, src=0)
    for st in wl.steps[:-1]:
        kv.plan(st.desc).close()
    batch = ny.Batch(wl.final.desc)
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, s.dtype, world)
    pred = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA)).bind(kv)
    slots, t_pred = None, 0.0
    t0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        plan = kv.plan(batch)
        if slots is None:
            slots = plan.slots()
        t_pred = pred.predict(batch)
        plan.rollback()
        plan.close()
    host_us = (time.perf_counter() - t0) * 1e6 / (args.warmup + args.steps)
    got = [None] * world
    if dist:
        dist.all_gather_object(got, (slots, len(uid[0])))
    else:
        got = [(slots, len(uid[0]))]
    if rank == 0:
        print(json.dumps({"impl": "host-only", "metric": METRIC, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "value": None, "world_size_seen": world,
                          "replicated_plans_equal": all(g == got[0] for g in got),
                          "unique_id_bytes": [g[1] for g in got], "host_step_us": host_us,
                          "predicted_launch_s": t_pred, "config": {"workload": wl.name,
                          "parallelism": f"kv-head shard x{world}"}}), flush=True)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    return "unknown"


def oracle_rows(wl, T, D):
    """The row sample both oracle legs time (cpu_baseline and --impl reference): 32 evenly
    spaced prefill rows and every decode row."""
    return list(range(0, T - D, max(1, (T - D) // 32))) + list(range(T - D, T))


def _oracle_pool(wl):
    from oracle.kvcache import KVPool
    s = wl.shape
    pool = KVPool(1, s.num_kv_heads, s.head_dim, s.block_size, wl.num_blocks, s.dtype)
    plan = None
    for st in wl.steps:
        plan = pool.plan(st.desc)
        pool.append(0, plan, st.k, st.v)
    return pool, plan


def cpu_baseline(wl, budget_s=20.0):
    """The fp64 oracle as it stands, on this host's cores, over a bounded row sample; timed
    with the BLAS pool at its default size and again at 1 thread."""
    from oracle import attention as OA
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # pragma: no cover
        threadpool_limits, threads = None, 1
    s = wl.shape
    pool, plan = _oracle_pool(wl)
    T = len(plan.rows)
    D = wl.final.desc.num_decode
    rows = oracle_rows(wl, T, D)

    def timed(budget):
        t0 = time.perf_counter()
        done = 0
        for r in rows:
            OA.hybrid_attention(pool, 0, plan, wl.final.q, s.num_q_heads, rows=[r])
            done += 1
            if time.perf_counter() - t0 > budget:
                break
        return done, time.perf_counter() - t0
    done, dt = timed(budget_s * 0.6)
    one = None
    if threadpool_limits is not None:
        with threadpool_limits(limits=1):
            d1, t1 = timed(budget_s * 0.4)
        one = {"value": d1 / t1, "unit": "tokens/s", "cores": 1, "rows": d1}
    return {"value": done / dt, "unit": "tokens/s", "cores": threads, "kind": "oracle",
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model(), "one_thread": one,
            "sample": f"{done} of {T} batch rows ({len(rows) - D} evenly spaced prefill rows + all {D} decode "
                      f"rows, all {s.num_q_heads} heads), fp64 numpy, {dt:.1f} s (the reference arm's sample)"}


def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm), rank 0 only."""
    if rank != 0:
        return
    from oracle import attention as OA
    wl = workload(args.config)
    s = wl.shape
    pool, plan = _oracle_pool(wl)
    T = len(plan.rows)
    D = wl.final.desc.num_decode
    sample = oracle_rows(wl, T, D)   # the cpu_baseline leg's sample, 8 rows per step, cycling
    per_step = 8
    pos = [0]

    def one():
        rows = sorted(sample[(pos[0] + i) % len(sample)] for i in range(per_step))
        pos[0] = (pos[0] + per_step) % len(sample)
        OA.hybrid_attention(pool, 0, plan, wl.final.q, s.num_q_heads, rows=rows)
        return len(rows)

    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    n = sum(one() for _ in range(args.steps))
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # pragma: no cover
        threads = 1
    v = n / dt
    out = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": wl.name, "step": f"fp64 oracle on {per_step} rows of the batch per step "
                      f"(cycling through the cpu_baseline sample: {len(sample)} rows)"},
           "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                            "sample": f"{per_step} random batch rows per step of {T}"},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def paper_context():
    """The paper's own published numbers with their hardware — context for
    the reader, not a target: they are full-model serving metrics on A100, not
    per-layer attention tokens/s.  Plus this repo's fig:chunk-perf analogue from the
    committed config-3 sweep, if present."""
    ctx = {"hardware": "NVIDIA A100 80 GB (Llama3-8B on 1 GPU; Qwen-7B TP2), P:364",
           "serving_capacity_vs_siloed_sarathi": "+32% (P:29, P:87)",
           "goodput_vs_sarathi_fcfs_edf": "1.5-2.4x / +20-40% (Azure-Code, P:446)",
           "ablation_capacity_qps": "EDF 2.75, +dynamic chunking 3.3, +eager relegation 3.6, +hybrid priority 3.65 "
                                    "(Llama3-8B, P:555-558)",
           "small_chunk_throughput": "28% lower full-model throughput at small chunks (P:71)"}
    fit = os.path.join(ROOT, "profiles", "predictor_fit.json")
    if os.path.exists(fit):
        try:
            r = json.load(open(fit)).get("chunk256_vs_2048_throughput_ratio")
            if r is not None:
                ctx["this_repo_attention_chunk256_vs_2048"] = round(float(r), 3)
        except (OSError, ValueError):
            pass
    return ctx


def main():
    args = parse()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args.gpus))
    rank, world, local, dist = dist_setup(args.gpus, args.host_only)
    if args.host_only:
        run_host_only(args, rank, world, dist)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import numpy as np
    import torch

    import paper_2503_22562_b200 as ny
    import workloads as W

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wl = workload(args.config)
    s = wl.shape
    hq, hkv = s.num_q_heads // world, s.num_kv_heads // world
    q0, k0 = rank * hq, rank * hkv
    fused = args.fused_append
    # the model's layer count (Llama-3-8B 32, Llama-3-70B 80), capped so the per-rank KV of all
    # layers fits in ~120 GB of HBM (config 4 at N = 1: 4.3 GB per layer -> 27 layers)
    per_layer = (wl.num_blocks + 64) * hkv * s.block_size * s.head_dim * 2 * s.elt_bytes
    L = args.layers if args.layers > 0 else min(32 if args.config == "l8b" else 80, max(1, int(120e9 // per_layer)))
    kv = ny.KVCache(L, s.num_q_heads, s.num_kv_heads, s.head_dim, wl.num_blocks + 64, block_size=s.block_size,
                    dtype=s.dtype, world_size=world, rank=rank, device=local)
    if args.tuning:
        kv.set_tuning(**{k: int(v) for k, v in (x.split("=") for x in args.tuning.split(","))})
    gather_fused = args.gather == "fused"
    if world > 1:
        uid = ny.get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        kv.comm_init(obj[0])
    elif gather_fused:
        kv.comm_init(ny.get_unique_id())

    def dev_bf16(a, lo, hi):
        return torch.from_numpy(np.ascontiguousarray(a[:, lo:hi]).view(np.int16)).to(dev).view(torch.bfloat16)

    # prefix fill (untimed): sequences pre-filled by the library's own append, every layer
    for st in wl.steps[:-1]:
        p = kv.plan(st.desc)
        kd, vd = dev_bf16(st.k, k0, k0 + hkv), dev_bf16(st.v, k0, k0 + hkv)
        for layer in range(L):
            kv.append(p, layer, kd, vd)
        torch.cuda.synchronize()
        p.close()
    fin = wl.final
    desc = fin.desc
    T = desc.num_rows
    q = dev_bf16(fin.q, q0, q0 + hq)
    k_new = dev_bf16(fin.k, k0, k0 + hkv)
    v_new = dev_bf16(fin.v, k0, k0 + hkv)
    o_full = torch.empty((s.num_q_heads, T, s.head_dim), dtype=torch.bfloat16, device=dev)
    lse_full = torch.empty((s.num_q_heads, T), dtype=torch.float32, device=dev)
    o = o_full[q0:q0 + hq]
    lse = lse_full[q0:q0 + hq]
    stream = torch.cuda.current_stream()
    window = kv.gather_window(T) if gather_fused else None
    last_win = {}

    # a8 predictor: fitted parameters from the config-3 sweep if committed, else roofline-shaped defaults
    fit_path = os.path.join(ROOT, "profiles", "predictor_fit.json" if args.config == "l8b" else
                            f"predictor_fit_{args.config}.json")
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, s.dtype, world)
    theta = list(ny.DEFAULT_THETA)   # the config-3 fit of round 2 (profiles/predictor_fit.json)
    if os.path.exists(fit_path):
        fj = json.load(open(fit_path))
        ok = fj.get("world", 1) == world and fj.get("config") == args.config and len(fj.get("theta", [])) == ny.NUM_PARAMS
        theta = fj["theta"] if ok else theta
    pred = ny.Predictor.from_params(cfg, theta)
    # a1 inputs: decodes carry Table 3 tiers; interactive ones are mid-stream
    DecodeQoS = ny.DecodeQoS
    tiers = desc.tiers()
    qos = []
    for j in range(desc.num_decode):
        tier = tiers[desc.num_prefill + j] % 3
        if tier == 0:
            qos.append(DecodeQoS(True, 0.0, slo_ttft=6.0, slo_tbt=0.05, next_token=40))
        else:
            qos.append(DecodeQoS(False, 0.0, slo_ttlt=600.0 if tier == 1 else 1800.0, est_remaining=400))
    qos_arr = ny.QoSArray(qos)
    batch = ny.Batch(desc)                              # marshalled once, reused every step
    dec_only = ny.Batch(W.BatchDesc(decode_seq=desc.decode_seq, decode_ctx=desc.decode_ctx))
    c_off = desc.prefill_offset[0] if desc.num_prefill else 0
    c_rem = desc.prefill_len[0] if desc.num_prefill else 0
    a1 = {}

    def a1_step():
        sl = qos_arr.min_slack(7.9)
        c, inf = pred.max_feasible_chunk(dec_only, c_off, c_rem, sl, 2048)
        a1["slack_s"], a1["chunk"], a1["infeasible"] = sl, c, inf

    # Per-launch events cost device time (~1-2 us each) and break the programmatic
    # launch overlap of append -> attention, so they bracket every EV_EVERY-th timed
    # step only; the attention roofline uses the mean over those launches.
    EV_EVERY = 4
    ev = [[tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(L)] if i % EV_EVERY == 0
          else None for i in range(args.steps)]

    def step(evs=None):
        a1_step()                                       # a1 (host)
        plan = kv.plan(batch, stream)                   # a2: once per iteration, all layers
        for layer in range(L):
            ev_ = evs[layer] if evs is not None else None   # events bracket every layer's launches
            if ev_ is not None:
                ev_[0].record(stream)
            if gather_fused:   # a4-a7 (a3-a7 with --fused-append) in ONE launch (niyama_attention_gather)
                if not fused:
                    kv.append(plan, layer, k_new, v_new, stream)
                if ev_ is not None:
                    ev_[1].record(stream)
                last_win["o"] = kv.attention_gather(plan, layer, q, window, k_new if fused else None,
                                                    v_new if fused else None, 0.0, stream)[0]
            elif fused:   # a3-a6 in ONE launch (niyama_append_attention)
                if ev_ is not None:
                    ev_[1].record(stream)
                kv.append_attention(plan, layer, k_new, v_new, q, o, lse, 0.0, stream)
            else:
                kv.append(plan, layer, k_new, v_new, stream)        # a3
                if ev_ is not None:
                    ev_[1].record(stream)
                kv.attention(plan, layer, q, o, lse, 0.0, stream)   # a4-a6
            if ev_ is not None:
                ev_[2].record(stream)
            if world > 1 and not gather_fused:
                kv.allgather_heads(plan, o_full, lse_full, stream)   # a7
            if ev_ is not None:
                ev_[3].record(stream)
        pred.predict(batch)                             # a8
        plan.rollback()                                 # replay the same batch next step (host only)
        plan.close()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    t_settle = time.time()
    while time.time() - t_settle < args.settle_s:
        for _ in range(20):
            step()
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    for i in range(args.steps):
        step(ev[i])
    host_issue_us = (time.perf_counter() - h0) * 1e6 / args.steps
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    attn_ms = [e[1].elapsed_time(e[2]) for es in ev if es is not None for e in es]
    append_ms = [e[0].elapsed_time(e[1]) for es in ev if es is not None for e in es]
    ag_ms = [e[2].elapsed_time(e[3]) for es in ev if es is not None for e in es]
    attn_avg_ms = sum(attn_ms) / len(attn_ms)
    ag_avg_ms = sum(ag_ms) / len(ag_ms)
    attn_q = [float(x) for x in np.percentile(np.array(attn_ms) * 1e3, [10, 50, 90])]
    attn_med_ms = attn_q[1] * 1e-3   # the roofline's launch time: median (robust to a throttled launch)
    per_rank = {"attention_us": [attn_med_ms * 1e3], "allgather_us": [ag_avg_ms * 1e3], "step_us": [ms / args.steps * 1e3]}
    if dist:
        t = torch.tensor([ms, attn_med_ms, ag_avg_ms], device=dev)
        allr = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
        per_rank = {"attention_us": [float(x[1]) * 1e3 for x in allr], "allgather_us": [float(x[2]) * 1e3 for x in allr],
                    "step_us": [float(x[0]) / args.steps * 1e3 for x in allr]}
        ms = max(float(x[0]) for x in allr)
        attn_med_ms = max(float(x[1]) for x in allr)

    # ---- e2e through the public API with host buffers (pinned), copies inside the
    # timed region.  Two buffer sets: the H2D of step i+1 (copy stream) and the
    # D2H of step i-1 (second copy stream) overlap step i's kernels.
    h_q = q.cpu().pin_memory()
    h_k = k_new.cpu().pin_memory()
    h_v = v_new.cpu().pin_memory()
    h_o = [torch.empty_like(o_full, device="cpu").pin_memory() for _ in range(2)]
    d_q = [torch.empty_like(q) for _ in range(2)]
    d_k = [torch.empty_like(k_new) for _ in range(2)]
    d_v = [torch.empty_like(v_new) for _ in range(2)]
    e_of = [torch.empty_like(o_full) for _ in range(2)]
    e_lf = [torch.empty_like(lse_full) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]      # inputs of buffer b landed
    ev_used = [torch.cuda.Event() for _ in range(2)]    # kernels of buffer b done (inputs free, output ready)
    ev_out = [torch.cuda.Event() for _ in range(2)]     # output of buffer b copied out
    for b_ in range(2):
        for e_ in (ev_used[b_], ev_out[b_]):
            e_.record(stream)

    ctr = [0]   # layers issued so far: buffer set = ctr & 1

    def e2e_step(i):
        a1_step()
        plan = kv.plan(batch, stream)
        for layer in range(L):   # each layer's Q/K/V arrive from the host, its O goes back
            b_ = ctr[0] & 1
            ctr[0] += 1
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_used[b_])
                d_q[b_].copy_(h_q, non_blocking=True)
                d_k[b_].copy_(h_k, non_blocking=True)
                d_v[b_].copy_(h_v, non_blocking=True)
                ev_in[b_].record(s_in)
            stream.wait_event(ev_in[b_])
            stream.wait_event(ev_out[b_])
            if gather_fused:
                if not fused:
                    kv.append(plan, layer, d_k[b_], d_v[b_], stream)
                wo, wl_ = kv.attention_gather(plan, layer, d_q[b_], window, d_k[b_] if fused else None,
                                              d_v[b_] if fused else None, 0.0, stream)
                e_of[b_].copy_(wo)     # the consumer reads the window before the next call (its contract)
                e_lf[b_].copy_(wl_)
            elif fused:
                kv.append_attention(plan, layer, d_k[b_], d_v[b_], d_q[b_], e_of[b_][q0:q0 + hq],
                                    e_lf[b_][q0:q0 + hq], 0.0, stream)
            else:
                kv.append(plan, layer, d_k[b_], d_v[b_], stream)
                kv.attention(plan, layer, d_q[b_], e_of[b_][q0:q0 + hq], e_lf[b_][q0:q0 + hq], 0.0, stream)
            if world > 1 and not gather_fused:
                kv.allgather_heads(plan, e_of[b_], e_lf[b_], stream)
            ev_used[b_].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_used[b_])
                h_o[b_].copy_(e_of[b_], non_blocking=True)
                ev_out[b_].record(s_out)
        pred.predict(batch)
        plan.rollback()
        plan.close()

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(s_in)
    for i in range(args.steps):
        e2e_step(i)
    for b_ in range(2):
        stream.wait_event(ev_out[b_])
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    ok = bool(torch.equal(h_o[(ctr[0] - 1) & 1], (last_win["o"] if gather_fused else o_full).cpu()))
    clocks.stop()
    h2d = (h_q.numel() + h_k.numel() + h_v.numel()) * 2 * L
    d2h = h_o[0].numel() * 2 * L

    B_kv, F = algorithmic(wl, hq, hkv)
    hbm_peak, tf_peak, peak_src = peaks()
    attn_s = attn_med_ms * 1e-3
    achieved = B_kv / attn_s / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        pj = json.load(open(prof))
        traffic = pj.get(f"{args.config}-g{world}", {}).get("dram_bytes_per_launch")
    value = T * L * args.steps / (ms * 1e-3)   # layer-tokens: each of the L layers attends the T rows
    out = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: seeded PCG64, Q/K/V ~ N(0,1) rounded to bf16; decode ctx ~ U{1..4096} (seed 0)",
        "config": {"workload": wl.name, "Hq": s.num_q_heads, "Hkv": s.num_kv_heads, "head_dim": s.head_dim,
                   "block_size": s.block_size, "chunk": sum(desc.prefill_len),
                   "chunk_offset": desc.prefill_offset[0] if desc.num_prefill else 0,
                   "num_decode": desc.num_decode, "sum_ctx": int(sum(desc.decode_ctx)), "T": T,
                   "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
                   "layers": L,
                   "l2": f"inputs larger than L2 ({B_kv / 1e6:.0f} MB KV read per layer per GPU vs 126 MB L2; "
                         f"every layer has its own KV)",
                   "step": (f"one iteration: a1 slack+chunk, a2 plan (once), then per layer x{L}: " +
                            ("a3-a6 ONE launch (append inside the attention)" if fused else
                             "a3 append, a4-a6 fused attention")) +
                           (", a7 all-gather INSIDE the attention launch (symmetric-window stores + flag barrier)"
                            if gather_fused else ", a7 NCCL all-gather" if world > 1 else "") +
                           "; a8 predict; value = T x layers / step time",
                   **({"tuning": args.tuning} if args.tuning else {})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "traffic_source": "stored: dram__bytes_read.sum + dram__bytes_write.sum of this launch from one "
                                       "ncu --set full capture (profiles/ncu_traffic.json), not measured in this run",
                     "kernel": "hybrid_attn_bf16_kernel" + (" (incl. the KV append)" if fused else "") +
                               (" (incl. the head all-gather)" if gather_fused else ""),
                     "algorithmic_bytes_per_launch": B_kv,
                     "launch_us": attn_med_ms * 1e3, "launch_stat": "median over the event-bracketed launches (rank max)",
                     "peak_source": peak_src,
                     "tensor_frac": F / attn_s / (tf_peak * 1e12),
                     "t_roof_us": max(F / (tf_peak * 1e12), B_kv / (hbm_peak * 1e9)) * 1e6},
        "attn_tokens_per_s": T / attn_s,
        "step_breakdown_us": {"append": 1e3 * sum(append_ms) / len(append_ms), "attention": attn_med_ms * 1e3,
                              "allgather": ag_avg_ms * 1e3,
                              "other_per_layer": ms / args.steps / L * 1e3 - attn_med_ms * 1e3
                                                 - 1e3 * sum(append_ms) / len(append_ms),
                              "step": ms / args.steps * 1e3, "per_layer": ms / args.steps / L * 1e3,
                              "host_issue": host_issue_us,
                              "note": "append/attention/allgather: every layer's launches of the event-bracketed steps"},
        "attention_launch_us": {"p10": attn_q[0], "median": attn_q[1], "p90": attn_q[2], "mean": attn_avg_ms * 1e3,
                                "samples": len(attn_ms)},
        "per_rank": per_rank,
        "e2e": {"value": T * L * args.steps / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "output_matches_device_run": ok,
                "pipeline": "per layer: its Q/K/V H2D and O D2H on copy streams, 2 buffer sets, overlapping the "
                            "neighbouring layers' kernels"},
        "gpu_launches": (1 if fused else 2) * L * args.steps,
        "timing_note": (f"attention/append/all-gather launch times from events around every layer's launches on "
                        f"every {EV_EVERY}th timed step (those steps lose the append -> attention programmatic "
                        "overlap); the roofline uses their median (rank max; mean, p10, p90 in attention_launch_us); "
                        "the append interval of layer 0 includes the wait for the plan's upload"),
        "clocks": clocks.summary(t_settle, t_wall1),
        "a1": a1,
        "a8": {"predicted_attention_us": pred.predict(batch) * 1e6, "measured_attention_us": attn_med_ms * 1e3,
               "rel_err": pred.predict(batch) * 1e3 / attn_med_ms - 1.0,
               "note": "the event model fitted on flushed single launches (profiles/predictor_fit.json) vs the "
                       "mean launch inside the bench step (not flushed: inputs larger than L2)"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl)
    out["paper_context"] = paper_context()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

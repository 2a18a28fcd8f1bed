"""GPU diagnostics: run small cases one by one and print errors vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from tests.gpu_harness import Run, oracle_for, to_host_f64, errors

def case(name, wl):
    t0 = time.time()
    try:
        r = Run(wl)
        o, lse = r.attention()
    except Exception as e:
        print(f"[{name}] EXC {e}", flush=True); return
    _, plan, O, L = oracle_for(wl)
    og = to_host_f64(o, wl.shape.dtype)
    ma, rl = errors(og, O)
    lg = lse.cpu().numpy()
    dl = np.nanmax(np.abs(lg - L))
    P = wl.final.desc.num_rows - wl.final.desc.num_decode
    per_row = np.nanmax(np.abs(og - O), axis=(0, 2))
    bad = np.where(~(per_row <= 2e-2))[0]
    print(f"[{name}] T={og.shape[1]} prefill_rows={P} max_abs={ma:.3e} rel_l2={rl:.3e} dlse={dl:.3e} "
          f"bad_rows={len(bad)} first_bad={bad[:10].tolist()} ({time.time()-t0:.1f}s)", flush=True)
    if len(bad):
        r0 = bad[0]
        h = int(np.nanargmax(np.nanmax(np.abs(og[:, r0] - O[:, r0]), axis=1)))
        print("   head", h, "gpu", og[h, r0, :6], "ref", O[h, r0, :6], "lse", lg[h, r0], L[h, r0], flush=True)

which = sys.argv[1:] or ["all"]
S = W.L8B
if "all" in which or "dec" in which:
    case("decode-only-short", W.hybrid(S, "d", prefill_offset=0, chunk=0, decode_ctx=[1, 5, 16, 17, 40], seed=1))
    case("decode-only-long", W.hybrid(S, "d2", prefill_offset=0, chunk=0, decode_ctx=[3000, 700, 129], seed=2))
if "all" in which or "pre" in which:
    case("prefill-o0-c128", W.hybrid(S, "p", prefill_offset=0, chunk=128, decode_ctx=[], seed=3))
    case("prefill-o0-c32", W.hybrid(S, "p", prefill_offset=0, chunk=32, decode_ctx=[], seed=3))
    case("prefill-o100-c77", W.hybrid(S, "p", prefill_offset=100, chunk=77, decode_ctx=[], seed=4))
    case("prefill-o1536-c512", W.hybrid(S, "p", prefill_offset=1536, chunk=512, decode_ctx=[], seed=5))
if "all" in which or "mix" in which:
    case("mixed", W.random_hybrid(S, seed=0, num_prefill=2, max_chunk=300, num_decode=9, max_ctx=900))
if "all" in which or "f32" in which:
    case("tiny-f32", W.config1_tiny())

"""A/B timing of library variants (tools/build_variant.py) on a few workloads.

    python tools/ab.py base pf0 pf2 ...      ("base" = the in-tree libniyama.so)
Each variant runs in its own process (NIYAMA_LIB_PATH picks the library)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = os.environ.get("AB_CASES", "prefill,mixed,l70b,decode")

CHILD = r'''
import os, sys
sys.path.insert(0, os.path.join(%r, "tools")); sys.path.insert(0, %r)
import workloads as W
from kbench import time_it
cases = %r.split(",")
for c in cases:
    if c == "prefill":
        time_it(W.hybrid(W.L8B, "prefill-only-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2))
    elif c == "prefill70":
        time_it(W.hybrid(W.L70B, "l70b-prefill-only-c2048-o6144", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4), reps=10)
    elif c.startswith("prefill_b"):
        import dataclasses
        B = int(c[len("prefill_b"):])
        time_it(W.hybrid(dataclasses.replace(W.L8B, block_size=B), f"prefill-only-c512-o1536-B{B}", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2))
    elif c.startswith("prefill70_b"):
        import dataclasses
        B = int(c[len("prefill70_b"):])
        time_it(W.hybrid(dataclasses.replace(W.L70B, block_size=B), f"l70b-prefill-only-B{B}", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4), reps=10)
    elif c == "mixed":
        time_it(W.config2_l8b())
    elif c == "decode":
        time_it(W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2))
    elif c == "l70b":
        time_it(W.config4_l70b(), reps=10)
'''

for tag in sys.argv[1:]:
    env = dict(os.environ)
    if tag != "base":
        env["NIYAMA_LIB_PATH"] = os.path.join(ROOT, "paper_2503_22562_b200", "_build", "variants", f"libniyama_{tag}.so")
    print(f"### {tag}", flush=True)
    subprocess.run([sys.executable, "-c", CHILD % (ROOT, ROOT, CASES)], env=env, check=False)

"""Prefill-CTA share sweep on config 4 (L70B c2048 o6144 + 128 x 8192): launch time vs
NIYAMA_PREFILL_CTAS (diagnostic for the CTA split at g = 8)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402

caps = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 64, 80, 96, 112, 128]
for cap in caps:
    env = dict(os.environ)
    if cap:
        env["NIYAMA_PREFILL_CTAS"] = str(cap)
    import subprocess
    code = ("import sys; sys.path.insert(0, 'tools'); sys.path.insert(0, '.'); import workloads as W; "
            "from kbench import time_it; time_it(W.config4_l70b(), reps=10)")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"cap={cap:3d}", r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:], flush=True)

"""Prefill-CTA share sweep on config 4 (L70B c2048 o6144 + 128 x 8192): launch time vs
the niyama_tuning prefill_ctas cap (diagnostic for the CTA split at g = 8)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402

from kbench import time_it  # noqa: E402

caps = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 64, 80, 96, 112, 128]
for cap in caps:
    print(f"cap={cap:3d}", end=" ", flush=True)
    time_it(W.config4_l70b(), reps=10, tuning={"prefill_ctas": cap})

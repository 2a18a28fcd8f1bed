import sys; sys.path.insert(0,"tools"); sys.path.insert(0,".")
import workloads as W
from kbench import time_it
for wl in (W.hybrid(W.L70B, "l70b-prefill-c2048-o6144", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4),
           W.hybrid(W.L8B, "l8b-prefill-c2048-o2048", prefill_offset=2048, chunk=2048, decode_ctx=[], seed=4)):
    for cap in (148, 111, 74, 37):
        print(f"cap={cap:3d}", end=" "); time_it(wl, reps=10, tuning=dict(grid_cap=cap))

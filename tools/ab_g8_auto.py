import os, sys
sys.path.insert(0, '/root/repo/tools'); sys.path.insert(0, '/root/repo')
import workloads as W
from kbench import time_it
wl = W.config4_l70b()
for tun in (dict(), dict(decode_path=3), dict(prefill_pairs=2), dict(), dict(decode_path=3), dict(prefill_pairs=2)):
    print(tun or "auto", end=" ")
    time_it(wl, reps=20, tuning=tun)

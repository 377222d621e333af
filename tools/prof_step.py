"""Config-4 hybrid steps with per-section timings and device counters (profiling helper;
also the command ncu wraps: `ncu -k regex:fill_kernel -s 3 -c 1 python tools/prof_step.py`)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nh = int(sys.argv[2]) if len(sys.argv) > 2 else 4
f = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
wl = inputs.config(cfg, f=f)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w - 1):
    rom.step()
rom.sync()
every = int(sys.argv[4]) if len(sys.argv) > 4 else 1
for k in range(nh):
    rom.profile(True)
    rom.step()
    sec = rom.profile_read()
    cnt = rom.debug_counters(21)
    cnt = cnt[:16] + cnt[16:21]
    if k % every == 0 or k == nh - 1:
      print(f"hybrid {k}: " + " ".join(f"{n}={v[0]:.3f}" for n, v in sec.items() if v[1]), "counters", cnt, flush=True)
      t = rom.debug_timers(64)
      ts = [x for x in t[40:64] if x > 0]
      print("  sets us: " + " ".join("%.1f" % ((ts[i + 1] - ts[i]) / 1000) for i in range(len(ts) - 1) if ts[i + 1] > ts[i]), flush=True)
      d = [(t[i + 1] - t[i]) / 1000 for i in range(39) if t[i + 1] > t[i] and t[i] > 0 and t[i + 1] - t[i] < 1e8]
      tt = rom.debug_timers(96)
      sv = [x for x in tt[64:80] if x > 0]
      print("  solve us: " + " ".join("%.1f" % ((sv[i + 1] - sv[i]) / 1000) for i in range(len(sv) - 1)), flush=True)
      print("  filter us: prologue %.1f sweeps %s" % (d[0] if d else -1, " ".join("%.1f" % x for x in d[1:])), flush=True)
rom.sync()

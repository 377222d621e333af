"""Window-Gram (H10 / K11) timing through hrom_gram: C = (S - rho)^T (S - rho) over `rows` rows of
`ncol` plain fp64 columns on the FP64 tensor cores.  Reports ms, the symmetric flop count
rows * ncol * (ncol + 1) per second and its fraction of the measured DMMA peak
(profiles/r1_dmma_peak.json, 37.1 TF/s at 1965 MHz).

python tools/gram_bench.py --rows 67108864 --ncol 129     (config 5: 4096^2 x 4 vars, w = 128)
python tools/gram_bench.py --rows 16777216 --ncol 65      (config 4 re-base: 2048^2 x 4, w = 64)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM

PEAK = 37.107  # TF/s, tools/dmma_peak.cu (profiles/r1_dmma_peak.json)

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16777216)
ap.add_argument("--ncol", type=int, default=65)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--check", action="store_true", help="compare with a cuBLAS DGEMM of the same shift")
args = ap.parse_args()

wl = inputs.Workload("gram", dim=2, nx=64, ny=64, w=8, r=4)
rom = HybridROM(wl)
g = torch.Generator(device="cuda").manual_seed(5)
S = torch.rand((args.ncol, args.rows), dtype=torch.float64, device="cuda", generator=g) + 0.5
rho = torch.rand(args.rows, dtype=torch.float64, device="cuda", generator=g) + 0.5
for _ in range(2):
    C = rom.gram(S, rho)
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    C = rom.gram(S, rho)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
fl = args.rows * args.ncol * (args.ncol + 1)
out = {"rows": args.rows, "ncol": args.ncol, 
       "ms_best": ms, "ms_all": ts, "tflops_symmetric": fl / ms / 1e9, "frac_dmma_peak": fl / ms / 1e9 / PEAK}
if args.check:
    X = S - rho
    Cr = X @ X.T
    out["max_rel_err_vs_dgemm"] = float((C - Cr).abs().max() / Cr.abs().max())
print(json.dumps(out))

"""Algorithm-1 accuracy / cost metrics per config and full-HDM period z.

python tools/algorithm1_metrics.py [--configs 1,2,3] [--z 0,10,4] [--out gpurun_out/a1_metrics.json]

For each config: the whole run (BASELINE.json step counts; config 3 capped by --max-steps)
beside a full-HDM reference trajectory; reports e-bar, e at the last step, s-bar, s-bar*,
p-bar, t_R, t_H and S = t_H / t_R (paper_2301_01718_b200/algorithm1.py).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_01718_b200 import algorithm1 as A1  # noqa: E402
from paper_2301_01718_b200 import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--z", default="0,10,4")
    ap.add_argument("--max-steps", type=int, default=300)
    ap.add_argument("--out", default="gpurun_out/a1_metrics.json")
    args = ap.parse_args()
    out = {"device": torch.cuda.get_device_name(0), "runs": []}
    for cfg in [int(x) for x in args.configs.split(",")]:
        wl = inputs.config(cfg)
        steps = min(wl.steps, args.max_steps)
        for z in [int(x) for x in args.z.split(",")]:
            t0 = time.perf_counter()
            m = A1.run(wl, steps=steps, z=z)
            s = m.summary()
            s.update({"config": cfg, "workload": wl.name, "N": wl.N, "f": wl.f, "w": wl.w, "r": wl.r,
                      "wall_s": time.perf_counter() - t0,
                      "e_every_10": [m.e[i] for i in range(9, len(m.e), 10)]})
            out["runs"].append(s)
            print(json.dumps({k: v for k, v in s.items() if k != "e_every_10"}), flush=True)
            os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
            json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""Copy / summarise the GPU evidence of a round into profiles/ (tracked).

python tools/make_profiles.py r1
  gpurun_out/launches.csv      (ncu --metrics gpu__time_duration.sum --nvtx-include timed/ of bench.py)
  gpurun_out/fill_full.ncu-rep (ncu --set full of the fill kernel inside bench.py's timed region)
  gpurun_out/bench_default.json
-> profiles/<tag>_launches.csv, <tag>_launch_summary.txt, <tag>_fill_ncu_full.txt,
   <tag>_bench.json, fill_traffic.json
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launch_summary(path, steps):
    lines = open(path).read().splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    ki, vi, gi, bi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        n = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        a = agg.setdefault(n, [0, 0.0, r[gi], r[bi]])
        a[0] += 1
        a[1] += float(r[vi]) / 1e6
    tot = sum(a[1] for a in agg.values())
    out = io.StringIO()
    out.write(f"# ncu launch list of bench.py's timed region ({steps} hybrid steps, serialised, cold-cache)\n")
    out.write(f"# total {tot / steps:.3f} ms/step over {sum(a[0] for a in agg.values())} launches\n")
    out.write(f"{'kernel':44s} {'launches':>8s} {'ms/step':>8s} {'share':>6s}  grid x block\n")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"{n[:44]:44s} {a[0]:8d} {a[1] / steps:8.3f} {a[1] / tot:6.3f}  {a[2]} x {a[3]}\n")
    return out.getvalue(), agg, tot


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main(tag, steps=3):
    os.makedirs(PROF, exist_ok=True)
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(PROF, f"{tag}_launches.csv"))
        txt, _, _ = launch_summary(lp, steps)
        open(os.path.join(PROF, f"{tag}_launch_summary.txt"), "w").write(txt)
        print(txt)
    rep = os.path.join(OUT, "fill_full.ncu-rep")
    if os.path.exists(rep):
        v, u = ncu_raw(rep)
        keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
        s = io.StringIO()
        s.write("# ncu --set full --clock-control none, fill kernel (H6 fill + indicator + H10 Gram row),\n")
        s.write("# first launch inside bench.py's timed region (config 4, f = 10 %)\n")
        for k in keys:
            if k in v:
                s.write(f"{k} = {v[k]} {u.get(k, '')}\n")
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                              capture_output=True, text=True).stdout
        s.write("\n" + summ)
        open(os.path.join(PROF, f"{tag}_fill_ncu_full.txt"), "w").write(s.getvalue())

        def to_bytes(key):
            val = float(v[key].replace(",", ""))
            unit = u.get(key, "byte").lower()
            return val * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)

        traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
        json.dump({"kernel": "fill_kernel", "dram_bytes_per_launch": traffic,
                   "source": f"profiles/{tag}_fill_ncu_full.txt (dram__bytes_read.sum + dram__bytes_write.sum)"},
                  open(os.path.join(PROF, "fill_traffic.json"), "w"), indent=1)
        print(s.getvalue())
    bp = os.path.join(OUT, "bench_default.json")
    if os.path.exists(bp):
        shutil.copy(bp, os.path.join(PROF, f"{tag}_bench.json"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")

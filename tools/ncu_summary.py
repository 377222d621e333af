"""Summarise an ncu report: key raw metrics + the hottest source lines (stall samples)."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        d[h] = (v, u)
    return d


def main(rep, nlines=12):
    d = raw(rep)
    print("kernel:", d.get("Kernel Name", ("?",))[0][:100])
    for k in KEYS:
        if k in d:
            print(f"  {k} = {d[k][0]} {d[k][1]}")
    stalls = sorted(((float(v[0]), k) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not k.endswith("not_issued") and v[0] not in ("", "n/a")), reverse=True)[:8]
    print("  top stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(v)}" for v, k in stalls))
    for view in ("cuda", "sass"):
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                             capture_output=True, text=True).stdout
        rows = [r for r in csv.reader(io.StringIO(out)) if r and r[0] != "Kernel Name"]
        print(f"  -- {view} view --")
        _top(rows, nlines)


def _top(rows, nlines):
    if rows:
        hdr = rows[0]
        try:
            i_src = hdr.index("Source")
            i_s = [i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All")][0]
        except (ValueError, IndexError):
            print("  (no source page)")
            return
        lines = []
        for r in rows[1:]:
            try:
                lines.append((float(r[i_s] or 0), r[0], r[i_src].strip()[:110]))
            except (ValueError, IndexError):
                pass
        tot = sum(x[0] for x in lines) or 1
        for s, ln, src in sorted(lines, reverse=True)[:nlines]:
            print(f"  {100*s/tot:5.1f}%  {ln}: {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)

"""Planted-mutation check of the oracle's seam-filter pins (VERDICT r1 "what's weak" 1).

Each mutant rewrites one line of oracle/sampling_filter.cpp, rebuilds liboracle.so and runs
tests/test_oracle_sampling_filter.py, which must FAIL; the original source is restored after
every mutant.  Mutants: the y-pass reads v instead of v' (P:424-432 applies S^y to the x-filtered
values), an absolute instead of relative eps_f stop (reading A23), a reversed 6 -> 4 -> 2 cascade.

python tools/oracle_mutants.py        (CPU only; ~10 s)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "sampling_filter.cpp")
MUTANTS = {
    "y-pass reads v": ("s += c[m + rad] * vp[var * G.N + (int64_t)G.iy(j + m) * G.nx + i];",
                       "s += c[m + rad] * v[var * G.N + (int64_t)G.iy(j + m) * G.nx + i];"),
    "absolute eps_f": ("maxdec = std::max(maxdec, (rold - rnew) / rold);", "maxdec = std::max(maxdec, (rold - rnew));"),
    "reversed cascade": ("const int order = p->filter_orders[oi];",
                         "const int order = p->filter_orders[p->n_filter_orders - 1 - oi];"),
}


def rebuild():
    sys.path.insert(0, ROOT)
    import oracle
    oracle.build(force=True)


def main():
    orig = open(SRC).read()
    results = {}
    try:
        for name, (a, b) in MUTANTS.items():
            assert orig.count(a) == 1, name
            open(SRC, "w").write(orig.replace(a, b))
            rebuild()
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                                os.path.join(ROOT, "tests", "test_oracle_sampling_filter.py")],
                               cwd=ROOT, capture_output=True, text=True)
            results[name] = "caught" if r.returncode != 0 else "SURVIVED"
            print(f"{name}: {results[name]} ({r.stdout.strip().splitlines()[-1]})")
    finally:
        open(SRC, "w").write(orig)
        rebuild()
    sys.exit(0 if all(v == "caught" for v in results.values()) else 1)


if __name__ == "__main__":
    main()

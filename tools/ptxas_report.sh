#!/bin/bash
# Per-kernel registers / spills of one csrc/*.cu file (sm_100a), demangled.
# usage: tools/ptxas_report.sh paper_2301_01718_b200/csrc/linalg.cu
f=${1:?file}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -c "$f" -o /tmp/ptxas_report.o -Xptxas -v 2>&1 | python3 -c "
import sys,re,subprocess
name=None
for line in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",line)
    if m: name=m.group(1); continue
    m=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores',line)
    if m and name: stack,spill=m.group(1),m.group(2); continue
    m=re.search(r'Used (\d+) registers',line)
    if m and name:
        dem=subprocess.run(['c++filt',name],capture_output=True,text=True).stdout.strip()
        dem=re.sub(r'hrom::\(anonymous namespace\)::','',dem)[:100]
        print(f'{m.group(1):>4} regs  stack {stack:>4} spill {spill:>4}  {dem}')
        name=None
"

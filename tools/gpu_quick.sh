#!/bin/bash
# quick GPU check after a kernel change: selected parity tests (PYTEST_K) + a short bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "${PYTEST_K:-full_step or masked or determinism or replay_parity or z1}" > gpurun_out/quick_tests.txt 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/quick_tests.txt)"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/quick_bench.json").read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"], 4), "full step ms", round(d["full_step"]["ms"], 4), "fill frac", round(d["roofline"]["frac"], 3))
print({k: round(v, 4) for k, v in d["section_ms_per_step"].items()})
PY

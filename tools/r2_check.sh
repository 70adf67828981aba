#!/bin/bash
# round-2 GPU check: all gpu tests, then a bench line per window setting
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "rel-L2|passed|failed|Error|error" | tail -60 > gpurun_out/r2_tests.log
tail -3 gpurun_out/r2_tests.log
for W in 1 0; do
  PATFFT_FP32_WINDOW=$W timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w$W.json 2> gpurun_out/bench_w$W.err || tail -5 gpurun_out/bench_w$W.err
  python - gpurun_out/bench_w$W.json <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[1], "ms/step %.3f  value %.3e vox/s  e2e %.2f ms" % (d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"] if d["e2e"] else -1))
for k, v in d["stages"].items():
    print("  %-12s %7.3f ms  %5.1f%%  %7.0f GB/s" % (k, v["ms"], 100 * v["share"], v["GBps"] or 0))
PY
done

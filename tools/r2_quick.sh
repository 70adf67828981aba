#!/bin/bash
# quick GPU check: parity subset (-k expression in $TESTS) + one bench line with stage times
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s ${TESTS:+-k "$TESTS"} 2>&1 | grep -E "rel-L2|passed|failed|Error|error" | tail -80 > gpurun_out/q_tests.log
tail -2 gpurun_out/q_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err || tail -5 gpurun_out/q_bench.err
python - gpurun_out/q_bench.json <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print("ms/step %.3f  value %.3e vox/s  e2e %.2f ms" % (d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"] if d["e2e"] else -1))
for k, v in d["stages"].items():
    print("  %-12s %7.3f ms  %5.1f%%  %7.0f GB/s" % (k, v["ms"], 100 * v["share"], v["GBps"] or 0))
PY

#!/bin/bash
# parity tests + one bench line with per-stage times (used with gpurun)
set -o pipefail
python /root/repo/paper_1501_02946_b200/_build.py > /dev/null || { echo BUILD FAILED; exit 1; }
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 || exit 1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err || { tail -20 gpurun_out/bench_q.err; exit 1; }
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_q.json"))
print("ms/step %.3f  value %.3e vox/s  e2e %.2f ms  stages-sum %.3f" % (d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"] if d["e2e"] else -1, sum(v["ms"] for v in d["stages"].values())))
for k, v in d["stages"].items():
    print("  %-12s %7.3f ms  %5.1f%%  %7.0f GB/s" % (k, v["ms"], 100 * v["share"], v["GBps"] or 0))
PY

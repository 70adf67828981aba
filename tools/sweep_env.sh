#!/bin/bash
# usage: sweep_env.sh "ENV1=a ENV2=b" "ENV1=c" ...   (bench cfg4 per setting; ms/step + stages)
mkdir -p gpurun_out
for setting in "$@"; do
  env $setting timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/sw.json 2> gpurun_out/sw.err || { echo "FAIL $setting"; tail -3 gpurun_out/sw.err; continue; }
  python - "$setting" <<'PY'
import json, sys
d = json.load(open("gpurun_out/sw.json"))
st = " ".join("%s=%.3f" % (k[:6], v["ms"]) for k, v in d["stages"].items())
e = d.get("e2e") or {}
print("%-40s ms/step %.4f  e2e %.2f (single %.2f)  %s" % (sys.argv[1], d["ms_per_step"], e.get("ms_per_step", -1), e.get("single_call_ms", -1), st))
PY
done

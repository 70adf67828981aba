#!/bin/bash
# Bench prebuilt library variants (paper_1501_02946_b200/var_*.so) against the default build.
# usage (on the GPU box): bash tools/variants.sh [bench args]; env VARIANT_ENVS="A=1;B=2 C=3" adds runtime-env runs
run() {
  local out
  out=$(PATFFT_LIB=$PWD/$1 timeout 300 env $3 python bench.py --steps 20 --warmup 3 --no-cpu-baseline "${@:4}" 2>/tmp/variant.err)
  if [ -z "$out" ]; then echo "$2: FAILED"; tail -3 /tmp/variant.err; return; fi
  echo "$out" | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%-40s %.3f ms  ' % ('$2', d['ms_per_step']) + '  '.join('%s %.3f' % (k, v['ms']) for k, v in d['stages'].items()))"
}
for lib in paper_1501_02946_b200/libpatfft_b200.so paper_1501_02946_b200/var_*.so; do
  [ -f "$lib" ] || continue
  run $lib "$(basename $lib)" "X=0" "$@"
  IFS=';' read -ra ENVS <<< "${VARIANT_ENVS:-}"
  for e in "${ENVS[@]}"; do run $lib "$(basename $lib) $e" "$e" "$@"; done
done

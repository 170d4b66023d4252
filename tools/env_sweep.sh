#!/bin/bash
# Sweep launch-plan environment knobs on the decode stack: one bench line per setting.
# usage: bash tools/env_sweep.sh "DECDEC_PREFETCH=1" "DECDEC_PREFETCH=8" ...  (run on the GPU box)
out=${OUT:-gpurun_out/env_sweep.txt}
: > "$out"
for setting in "$@"; do
  line=$(env $setting timeout 300 python bench.py ${BENCH_ARGS:-} --sweep-only --steps ${STEPS:-30} --warmup 5 \
         --sweep ${SWEEP:-0,21} 2>/dev/null | tail -1)
  python - "$setting" "$line" >> "$out" <<'PY'
import json, sys
s, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(f"{s:40s}", " ".join(f"k{k}={v['ms_per_step']*1e3/32:.2f}us/blk" for k, v in d["sweep"].items()))
except Exception as e:
    print(f"{s:40s} FAILED {e}: {line[:200]}")
PY
done
cat "$out"

# A/B of environment settings: decode-step sweep AND per-layer µs (no --sweep-only).  usage: T=tag SWEEP=0,21 bash tools/gpu_ab_layers.sh "A=1" "A=0"
set -x
mkdir -p gpurun_out
T=${T:-ab}
python paper_2412_20185_b200/build.py
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag
B="python bench.py --steps ${STEPS:-30} --warmup 5 --sweep ${SWEEP:-0,1,21} --no-cpu-baseline --no-w4 --no-unfused-extra --no-lut ${BARGS:-}"
for rep in 1 2; do
for s in "$@"; do
  env $s timeout 600 $B > gpurun_out/${T}_$(echo $s | tr '=, /.' '_____')_$rep.json 2>gpurun_out/${T}_err.txt || tail -5 gpurun_out/${T}_err.txt
done
done
python - "$T" <<'PY'
import json,glob,sys
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k: v["ms_per_step"] for k,v in d["sweep"].items()}, {c: [round(v[s]['us'],2) for s in v if s not in ('d_in','d_out')] for c,v in d.get('per_layer_us',{}).items()})
    except Exception as e: print(f, e)
PY
grep -i hugepages /proc/meminfo | head -3

set -x
mkdir -p gpurun_out
T=${T:-r2_s9}
python paper_2412_20185_b200/build.py
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o build/probe_pipes paper_2412_20185_b200/csrc/probe/probe_pipes.cu
for w in 4 8 16 32; do ./build/probe_pipes $w; done > gpurun_out/${T}_pipes.jsonl 2>&1
cat gpurun_out/${T}_pipes.jsonl
B="python bench.py --steps 30 --warmup 5 --sweep 0,4,21 --no-cpu-baseline --no-w4 --no-unfused-extra --no-lut --sweep-only"
for i in 1 2; do
timeout 600 $B > gpurun_out/${T}_coop1_$i.json 2>&1
DECDEC_COOP=0 timeout 600 $B > gpurun_out/${T}_coop0_$i.json 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2_s9_coop*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k: v["ms_per_step"] for k,v in d["sweep"].items()})
    except Exception as e: print(f, e)
PY

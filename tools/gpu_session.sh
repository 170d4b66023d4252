set -x
mkdir -p gpurun_out
python paper_2412_20185_b200/build.py
T=r2_s7
export DECDEC_PARITY_REPORT=gpurun_out/${T}_parity_report.json
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1; tail -3 gpurun_out/${T}_pytest.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --kernel-name kns=decdec --print-limit 50 python tools/sanitize_run.py > gpurun_out/${T}_san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/${T}_san_$tool.txt
done
B="python bench.py --steps 20 --warmup 5 --sweep 0,4,21 --no-cpu-baseline --no-w4 --no-unfused-extra --no-lut --sweep-only"
timeout 600 $B > gpurun_out/${T}_coop1.json 2>&1
DECDEC_COOP=0 timeout 600 $B > gpurun_out/${T}_coop0.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2_s7_coop*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k: v["ms_per_step"] for k,v in d["sweep"].items()})
    except Exception as e: print(f, e)
PY

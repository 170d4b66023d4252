set -x
mkdir -p gpurun_out
python paper_2412_20185_b200/build.py
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or k0 or stack or llama_shapes_all_columns or tp_shard" > gpurun_out/r2_s3_pytest16.txt 2>&1; tail -2 gpurun_out/r2_s3_pytest16.txt
DECDEC_GEMV_NC=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or k0 or stack or llama_shapes_all_columns or tp_shard" > gpurun_out/r2_s3_pytest8.txt 2>&1; tail -2 gpurun_out/r2_s3_pytest8.txt
B="python bench.py --steps 30 --warmup 5 --sweep 0 --kchunk 0 --no-cpu-baseline --no-w4 --no-unfused-extra"
timeout 600 $B > gpurun_out/r2_s3_nc16_pf.json 2>&1
DECDEC_L2PF_NEXT=0 timeout 600 $B > gpurun_out/r2_s3_nc16_nopf.json 2>&1
DECDEC_GEMV_NC=8 timeout 600 $B > gpurun_out/r2_s3_nc8_pf.json 2>&1
DECDEC_GEMV_NC=8 DECDEC_L2PF_NEXT=0 timeout 600 $B > gpurun_out/r2_s3_nc8_nopf.json 2>&1
DECDEC_OLD_GEMV=1 timeout 600 $B > gpurun_out/r2_s3_old.json 2>&1
timeout 300 python tools/trace_stack.py --kchunk 0 --blocks 4 > gpurun_out/r2_s3_trace_nc16.txt 2>&1
DECDEC_GEMV_NC=8 timeout 300 python tools/trace_stack.py --kchunk 0 --blocks 4 > gpurun_out/r2_s3_trace_nc8.txt 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2_s3_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["sweep"]["0"]["ms_per_step"], {k:v["0"]["us"] for k,v in d.get("per_layer_us",{}).items()})
    except Exception as e: print(f, e)
PY
sed -n 5,10p gpurun_out/r2_s3_trace_nc16.txt
sed -n 5,10p gpurun_out/r2_s3_trace_nc8.txt

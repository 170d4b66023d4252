set -x
mkdir -p gpurun_out
T=r2_s12
python paper_2412_20185_b200/build.py
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "speculative or every_dec or fused_selection or config1 or llama_shapes" > gpurun_out/${T}_pytest.txt 2>&1; tail -5 gpurun_out/${T}_pytest.txt
SWEEP=0,1,4,21 T=${T}_ab bash tools/gpu_ab.sh DECDEC_SPEC_KB=48 DECDEC_SPEC_KB=0 DECDEC_SPEC_KB=128 2>&1 | grep gpurun_out
python tools/trace_stack.py --kchunk 1 --blocks 2 > gpurun_out/${T}_trace_k1.txt 2>&1
python tools/trace_stack.py --kchunk 21 --blocks 2 > gpurun_out/${T}_trace_k21.txt 2>&1

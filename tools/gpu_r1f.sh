timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or llama or tp_shard or fused_sel or chunk" 2>&1 | tail -3 > gpurun_out/r1f_pytest.txt
OUT=gpurun_out/r1f_sweep.txt STEPS=100 SWEEP=0,21 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_XPF=1" "DECDEC_XPF=0" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_XPF=1" "DECDEC_XPF=0" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_XPF=1" "DECDEC_XPF=0"
timeout 300 python tools/trace_stack.py --kchunk 21 --blocks 2 > gpurun_out/r1f_trace_k21.txt 2>&1
timeout 300 python tools/trace_stack.py --kchunk 0 --blocks 2 > gpurun_out/r1f_trace_k0.txt 2>&1
cat gpurun_out/r1f_pytest.txt

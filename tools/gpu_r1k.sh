timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "select or fused or config1 or llama" 2>&1 | tail -3 > gpurun_out/r1k_pytest.txt
OUT=gpurun_out/r1k_sweep.txt STEPS=100 SWEEP=4,21 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_NDEC=64"
timeout 300 python tools/trace_stack.py --kchunk 21 --blocks 2 > gpurun_out/r1k_trace_k21.txt 2>&1
tail -3 gpurun_out/r1k_pytest.txt

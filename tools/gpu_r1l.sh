timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r1l_pytest.txt
OUT=gpurun_out/r1l_sweep.txt STEPS=100 SWEEP=4,21 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1"
timeout 300 python tools/trace_stack.py --kchunk 21 --blocks 2 > gpurun_out/r1l_trace_k21.txt 2>&1
tail -3 gpurun_out/r1l_pytest.txt

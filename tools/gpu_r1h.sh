timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r1h_pytest.txt
OUT=gpurun_out/r1h_sweep.txt STEPS=60 SWEEP=0,4,8,16,21,32 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1"
cat gpurun_out/r1h_pytest.txt

timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r1o_pytest.txt
OUT=gpurun_out/r1o_sweep.txt STEPS=100 SWEEP=4,21 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linear -s 24 -c 1 -o gpurun_out/r1o_gu_k21 python tools/profile_layer.py --shape 4096x28672 --kchunk 21 --iters 8 > gpurun_out/r1o_ncu_k21.log 2>&1
cat gpurun_out/r1o_pytest.txt gpurun_out/r1o_sweep.txt

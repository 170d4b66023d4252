OUT=gpurun_out/r1n_sweep.txt STEPS=100 SWEEP=0,4,21 bash tools/env_sweep.sh "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_serial.so" "DECDEC_LIB=build/libdecdec_rs1.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_serial.so" "DECDEC_LIB=build/libdecdec_rs1.so"
OUT=gpurun_out/r1n_sweep_phi3.txt STEPS=30 SWEEP=0 BENCH_ARGS="--model phi3_medium" bash tools/env_sweep.sh "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_rs1.so" "DECDEC_PLAN=8,2" "DECDEC_PLAN=16,2"
cat gpurun_out/r1n_sweep.txt

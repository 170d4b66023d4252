OUT=gpurun_out/r1m_sweep.txt STEPS=100 SWEEP=4,21 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1"
timeout 900 python bench.py --bits 4 --no-cpu-baseline > gpurun_out/r1m_bench_w4.json 2> gpurun_out/r1m_bench_w4.err
timeout 900 python bench.py --model phi3_medium --no-cpu-baseline --sweep 0,21 > gpurun_out/r1m_bench_phi3.json 2> gpurun_out/r1m_bench_phi3.err
cat gpurun_out/r1m_sweep.txt; tail -c 300 gpurun_out/r1m_bench_w4.json; tail -c 300 gpurun_out/r1m_bench_phi3.json; tail -3 gpurun_out/r1m_bench_phi3.err

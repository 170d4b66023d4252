timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r1i_pytest.txt
OUT=gpurun_out/r1i_sweep.txt STEPS=100 SWEEP=4,21 bash tools/env_sweep.sh "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1" "DECDEC_LIB=build/libdecdec_base.so" "DECDEC_X=1"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1i_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r1i_bench.json 2> gpurun_out/r1i_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_linear -c 640 --csv --log-file gpurun_out/r1i_launches.csv python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/r1i_pytest.txt gpurun_out/r1i_smoke.txt

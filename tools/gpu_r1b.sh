timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tp or stack" > gpurun_out/r1b_pytest_tp.txt 2>&1
timeout 300 python tools/trace_stack.py --kchunk 21 --blocks 2 > gpurun_out/r1b_trace_k21.txt 2>&1
timeout 300 python tools/trace_stack.py --kchunk 0 --blocks 2 > gpurun_out/r1b_trace_k0.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_linear -c 640 --csv --log-file gpurun_out/r1_launches.csv python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_launch_bench.log 2>&1
tail -3 gpurun_out/r1b_pytest_tp.txt

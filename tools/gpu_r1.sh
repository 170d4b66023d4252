set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1_launches.csv python bench.py --quick --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linear -s 24 -c 1 -o gpurun_out/r1_gu_k21 python tools/profile_layer.py --shape 4096x28672 --kchunk 21 --iters 8 > gpurun_out/r1_ncu_k21.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linear -s 24 -c 1 -o gpurun_out/r1_gu_k0 python tools/profile_layer.py --shape 4096x28672 --kchunk 0 --iters 8 > gpurun_out/r1_ncu_k0.log 2>&1
tail -3 gpurun_out/r1_pytest_gpu.txt; cat gpurun_out/r1_smoke.txt | tail -2; head -c 600 gpurun_out/r1_bench.json

timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "validation or tp" 2>&1 | tail -3 > gpurun_out/r1s_pytest.txt
timeout 1200 python bench.py --model llama3_70b --shard-of 8 --no-cpu-baseline --sweep 0,21 --steps 50 > gpurun_out/r1s_bench_70b_shard8.json 2> gpurun_out/r1s_bench_70b_shard8.err
timeout 900 python bench.py --model phi3_medium --shard-of 8 --no-cpu-baseline --sweep 0,21 --steps 50 > gpurun_out/r1s_bench_phi3_shard8.json 2> gpurun_out/r1s_bench_phi3_shard8.err
cat gpurun_out/r1s_pytest.txt; tail -c 400 gpurun_out/r1s_bench_70b_shard8.json; tail -3 gpurun_out/r1s_bench_70b_shard8.err; tail -c 300 gpurun_out/r1s_bench_phi3_shard8.json

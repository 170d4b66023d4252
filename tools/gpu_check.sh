timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/check_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --sweep 21 --no-cpu-baseline > gpurun_out/check_bench.json 2>gpurun_out/check_bench.err
cat gpurun_out/check_pytest.txt gpurun_out/check_smoke.txt; head -c 300 gpurun_out/check_bench.json

python paper_2412_20185_b200/build.py; mkdir -p gpurun_out; export DECDEC_PARITY_REPORT=gpurun_out/final_parity_report.json
# Round-end measurement set (run on the GPU box): GPU tests, smoke, bench + reference arm,
# ncu launch list, ncu --set full of the gu layer at k_chunk 0/21, stack timeline -> gpurun_out/final_*
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_full.txt 2>&1; tail -3 gpurun_out/final_pytest_full.txt > gpurun_out/final_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_linear -c 640 --csv --log-file gpurun_out/final_launches.csv python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linear -s 24 -c 1 -o gpurun_out/final_gu_k21 python tools/profile_layer.py --shape 4096x28672 --kchunk 21 --iters 8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_linear -s 24 -c 1 -o gpurun_out/final_gu_k0 python tools/profile_layer.py --shape 4096x28672 --kchunk 0 --iters 8 > /dev/null 2>&1
timeout 300 python tools/trace_stack.py --kchunk 21 --blocks 2 > gpurun_out/final_trace_k21.txt 2>&1
cat gpurun_out/final_pytest.txt gpurun_out/final_smoke.txt; head -c 400 gpurun_out/final_bench.json; echo; head -c 600 gpurun_out/final_bench_ref.json

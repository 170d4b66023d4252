set -x
mkdir -p gpurun_out
python paper_2412_20185_b200/build.py
T=${T:-r2_s8}
export DECDEC_PARITY_REPORT=gpurun_out/${T}_parity_report.json
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1; tail -3 gpurun_out/${T}_pytest.txt
timeout 300 python tools/concurrency_check.py > gpurun_out/${T}_conc.txt 2>&1; echo "conc rc=$?"; cat gpurun_out/${T}_conc.txt | tail -2
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --kernel-name kns=decdec --print-limit 50 python tools/sanitize_run.py > gpurun_out/${T}_san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/${T}_san_$tool.txt
done
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/${T}_bench.json

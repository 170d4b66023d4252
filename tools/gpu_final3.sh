# Round-end measurement set (session 3): tests, smoke, bench + reference, ncu launch list + full
# captures, trace, secondary bench lines, compute-sanitizer memcheck/racecheck -> gpurun_out/final_*
set -x
bash tools/gpu_final.sh
bash tools/gpu_final2.sh
for tool in memcheck racecheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --kernel-name kns=decdec --print-limit 50 python tools/sanitize_run.py > gpurun_out/final_san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/final_san_$tool.txt
done

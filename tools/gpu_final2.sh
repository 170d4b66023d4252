# Secondary bench lines: 4-bit (config 3), Phi-3 (config 4), rank 0 of 8 for 70B / Phi-3 (configs 4/5)
timeout 900 python bench.py --bits 4 --no-cpu-baseline > gpurun_out/final_bench_w4.json 2> /dev/null
timeout 900 python bench.py --model phi3_medium --no-cpu-baseline --sweep 0,21 > gpurun_out/final_bench_phi3.json 2> /dev/null
timeout 1200 python bench.py --model llama3_70b --shard-of 8 --no-cpu-baseline --sweep 0,21 --steps 50 > gpurun_out/final_bench_70b_shard8.json 2> /dev/null
timeout 900 python bench.py --model phi3_medium --shard-of 8 --no-cpu-baseline --sweep 0,21 --steps 50 > gpurun_out/final_bench_phi3_shard8.json 2> /dev/null
for f in w4 phi3 70b_shard8 phi3_shard8; do python -c "import json,sys; d=json.loads(open('gpurun_out/final_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], {k:v['tokens_per_s'] for k,v in d['sweep'].items()}, d['roofline']['frac'])"; done

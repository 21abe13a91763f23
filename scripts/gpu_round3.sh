timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/timeline.py --algo alsd > gpurun_out/timeline_alsd.txt 2>&1
timeout 300 python scripts/timeline.py --algo greedy > gpurun_out/timeline_greedy.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1
timeout 1200 python scripts/bench_configs.py --only c3,c4,c5 --reps 1 > gpurun_out/configs_c3_c5.jsonl 2> gpurun_out/configs_c3_c5.err
cat gpurun_out/timeline_*.txt gpurun_out/gemm_trace.txt; tail -c 1500 gpurun_out/bench_bf16.log; cat gpurun_out/configs_c3_c5.jsonl; tail -n 5 gpurun_out/configs_c3_c5.err

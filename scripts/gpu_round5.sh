timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_gpu.log
for a in alsd greedy; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/timeline_$a.txt 2>&1; done
timeout 600 python scripts/timeline.py --config c5 --algo aes --frames 60 > gpurun_out/timeline_c5.txt 2>&1
timeout 600 python scripts/timeline.py --config c3 --algo alsd --frames 100 > gpurun_out/timeline_c3.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
timeout 300 python scripts/gemm_trace.py 40 c5 > gpurun_out/gemm_trace_c5.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c3 > gpurun_out/gemm_trace_c3.txt 2>&1
cat gpurun_out/timeline_*.txt gpurun_out/gemm_trace*.txt

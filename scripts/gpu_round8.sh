timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
timeout 300 python scripts/gemm_trace.py 40 c5 > gpurun_out/gemm_trace_c5.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c3 > gpurun_out/gemm_trace_c3.txt 2>&1
cat gpurun_out/gemm_trace*.txt

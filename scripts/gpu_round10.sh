timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
cat gpurun_out/gemm_trace*.txt

timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gpu_check.py > gpurun_out/gpu_check.txt 2>&1; grep -v "mismatch=0" gpurun_out/gpu_check.txt | tail -n 20
timeout 300 python scripts/timeline.py --algo alsd > gpurun_out/timeline_alsd.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c3 > gpurun_out/gemm_trace_c3.txt 2>&1
cat gpurun_out/timeline_alsd.txt gpurun_out/gemm_trace*.txt

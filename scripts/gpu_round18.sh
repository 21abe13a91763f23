set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 30 gpurun_out/pytest_gpu.log | cut -c1-400
timeout 600 python scripts/gemm_trace.py 40 c5 > gpurun_out/gemm_trace_c5.txt 2>&1; tail -n 5 gpurun_out/gemm_trace_c5.txt
timeout 1200 python scripts/timeline.py --config c5 --algo aes --frames 60 > gpurun_out/timeline_c5.txt 2>&1; head -6 gpurun_out/timeline_c5.txt

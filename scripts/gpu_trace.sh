set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
cat gpurun_out/gemm_trace.txt

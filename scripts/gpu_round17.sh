set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gpu_check.py > gpurun_out/gpu_check.txt 2>&1; tail -n 1 gpurun_out/gpu_check.txt
for a in alsd greedy; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/timeline_$a.txt 2>&1; echo "== $a"; head -6 gpurun_out/timeline_$a.txt; done
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1; tail -n 3 gpurun_out/gemm_trace.txt

set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gpu_check.py > gpurun_out/gpu_check.txt 2>&1; grep -v "mismatch=0" gpurun_out/gpu_check.txt | tail -n 12
TBEAM_BODY_PAIRS=1 timeout 300 python scripts/timeline.py --algo alsd > gpurun_out/timeline_alsd_p1.txt 2>&1
timeout 300 python scripts/timeline.py --algo alsd > gpurun_out/timeline_alsd.txt 2>&1
cat gpurun_out/timeline_alsd_p1.txt gpurun_out/timeline_alsd.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log | cut -c1-1500
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
tail -n 4 gpurun_out/gemm_trace.txt

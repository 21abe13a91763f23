set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gpu_check.py > gpurun_out/gpu_check.txt 2>&1; grep -v "mismatch=0" gpurun_out/gpu_check.txt | tail -n 20
for a in alsd greedy; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/timeline_$a.txt 2>&1; done
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1
cat gpurun_out/timeline_*.txt gpurun_out/gemm_trace.txt; tail -c 1200 gpurun_out/bench_bf16.log

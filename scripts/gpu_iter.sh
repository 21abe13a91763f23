# one build -> measure iteration on the GPU box: parity, round timeline, select
# phase trace, and the configs named in $CONFIGS (default c1,c2)
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/it/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it/pytest_gpu.log
for a in alsd greedy; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/it/timeline_$a.txt 2>&1; done
timeout 300 python scripts/gemm_trace.py > gpurun_out/it/gemm_trace.txt 2>&1
timeout 900 python scripts/bench_configs.py --only ${CONFIGS:-c1,c2} > gpurun_out/it/configs.jsonl 2> gpurun_out/it/configs.err
tail -2 gpurun_out/it/pytest_gpu.log; cat gpurun_out/it/timeline_*.txt gpurun_out/it/gemm_trace.txt; cut -c1-330 gpurun_out/it/configs.jsonl; tail -3 gpurun_out/it/configs.err

set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 600 python scripts/gemm_trace.py 40 c5 > gpurun_out/gemm_trace_c5.txt 2>&1
cat gpurun_out/gemm_trace_c5.txt
timeout 2000 python scripts/bench_configs.py --only c4,c5 --reps 1 > gpurun_out/configs_c4_c5.jsonl 2> gpurun_out/configs_c4_c5.err
cat gpurun_out/configs_c4_c5.jsonl | cut -c1-700; tail -n 3 gpurun_out/configs_c4_c5.err

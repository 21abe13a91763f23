# configs sweep + ncu launch list + full captures + phase traces
timeout 1500 python scripts/bench_configs.py --only c1,c2,c3,c4 > gpurun_out/configs_c1_c4.jsonl 2> gpurun_out/configs_c1_c4.err
timeout 300 python scripts/gemm_trace.py 100 > gpurun_out/gemm_trace.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bf16_alsd_T40.csv python scripts/profile_decode.py --frames 40 --reps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 40 -c 3 -o gpurun_out/prof_joint python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu_full_joint.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 40 -c 2 -o gpurun_out/prof_select python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu_full_select.log 2>&1
timeout 2400 python scripts/bench_configs.py --only c5 --reps 1 > gpurun_out/configs_c5.jsonl 2> gpurun_out/configs_c5.err
cat gpurun_out/configs_c1_c4.jsonl gpurun_out/configs_c5.jsonl gpurun_out/gemm_trace.txt; tail -5 gpurun_out/*.err gpurun_out/ncu_*.log

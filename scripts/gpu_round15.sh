set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gpu_check.py > gpurun_out/gpu_check.txt 2>&1; tail -n 1 gpurun_out/gpu_check.txt
for a in alsd greedy aes; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/timeline_$a.txt 2>&1; echo "== $a"; head -6 gpurun_out/timeline_$a.txt; done
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -c 4000 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bf16_alsd_T40.csv python scripts/profile_decode.py --frames 40 --reps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_fk -s 60 -c 3 -o gpurun_out/prof_fk python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu_full_fk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 30 -c 2 -o gpurun_out/prof_select python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu_full_select.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_bf16_alsd_T40.csv

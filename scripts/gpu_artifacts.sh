# full measurement pass for profiles/: bench, configs, timelines, ncu
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/art
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/art/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/art/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/art/bench.json 2> gpurun_out/art/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/art/bench_reference.json 2>&1
for a in alsd aes greedy; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/art/timeline_$a.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/art/launches_alsd_T40.csv python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/art/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/art/launches_alsd_T40.csv > gpurun_out/art/launches_alsd_T40.summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_fk -s 60 -c 3 -o gpurun_out/art/prof_fk python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/art/ncu_full_fk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 30 -c 2 -o gpurun_out/art/prof_select python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/art/ncu_full_select.log 2>&1
timeout 1500 python scripts/bench_configs.py --only c1,c2,c3,c4 > gpurun_out/art/configs_c1_c4.jsonl 2> gpurun_out/art/configs_c1_c4.err
timeout 1200 python scripts/timeline.py --config c5 --algo aes --frames 60 > gpurun_out/art/timeline_c5.txt 2>&1
timeout 2000 python scripts/bench_configs.py --only c5 --reps 1 > gpurun_out/art/configs_c5.jsonl 2> gpurun_out/art/configs_c5.err
cat gpurun_out/art/launches_alsd_T40.summary.txt; head -c 600 gpurun_out/art/bench.json; echo; cat gpurun_out/art/configs_c1_c4.jsonl gpurun_out/art/configs_c5.jsonl | cut -c1-400; tail -n 3 gpurun_out/art/*.err

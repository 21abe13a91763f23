set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -c 3000 gpurun_out/bench.log
for a in alsd greedy; do timeout 300 python scripts/timeline.py --algo $a > gpurun_out/timeline_$a.txt 2>&1; done
cat gpurun_out/timeline_*.txt
timeout 1500 python scripts/bench_configs.py --only c1,c2,c3,c4 > gpurun_out/configs_c1_c4.jsonl 2> gpurun_out/configs_c1_c4.err
cat gpurun_out/configs_c1_c4.jsonl; tail -n 3 gpurun_out/configs_c1_c4.err

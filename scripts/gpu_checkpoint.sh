# checkpoint: parity, the bench line, every BASELINE config
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/cp
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/cp/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cp/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/cp/bench.json 2> gpurun_out/cp/bench.err
timeout 1500 python scripts/bench_configs.py --only c1,c2,c3,c4 > gpurun_out/cp/configs_c1_c4.jsonl 2> gpurun_out/cp/configs_c1_c4.err
timeout 2000 python scripts/bench_configs.py --only c5 --reps 1 > gpurun_out/cp/configs_c5.jsonl 2> gpurun_out/cp/configs_c5.err
tail -1 gpurun_out/cp/pytest_gpu.log; tail -1 gpurun_out/cp/bench.json | cut -c1-700; cat gpurun_out/cp/configs_*.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'],d['algo'],'K',d['beam'],'rtfx %.0f'%d['rtfx'],'greedy %.0f'%d['greedy_rtfx'],'ratio %.2f'%d['beam_greedy_time_ratio'],'rounds',d['rounds'])"

mkdir -p gpurun_out/r2j
D=gpurun_out/r2j
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
for i in 1 2; do
timeout 120 python scripts/timeline.py --algo alsd > $D/tl_alsd_$i.txt 2>&1
timeout 120 python scripts/timeline.py --algo greedy > $D/tl_greedy_$i.txt 2>&1
done
timeout 300 python scripts/gemm_trace.py 100 > $D/trace.txt 2>&1
timeout 900 python scripts/bench_configs.py --only c3,c4 --reps 2 > $D/configs.jsonl 2>&1

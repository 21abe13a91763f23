mkdir -p gpurun_out/r2o
D=gpurun_out/r2o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
for i in 1 2; do
timeout 120 python scripts/timeline.py --algo alsd > $D/tl_alsd_mixed_$i.txt 2>&1
TBEAM_GATES_MIXED=0 timeout 120 python scripts/timeline.py --algo alsd > $D/tl_alsd_plain_$i.txt 2>&1
timeout 120 python scripts/timeline.py --algo greedy > $D/tl_greedy_mixed_$i.txt 2>&1
done
timeout 300 python scripts/timeline.py --config c3 --algo aes --frames 100 > $D/tl_c3_mixed.txt 2>&1
TBEAM_GATES_MIXED=0 timeout 300 python scripts/timeline.py --config c3 --algo aes --frames 100 > $D/tl_c3_plain.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err

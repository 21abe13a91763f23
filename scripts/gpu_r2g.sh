mkdir -p gpurun_out/r2g
D=gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
for i in 1 2; do
timeout 120 python scripts/timeline.py --algo alsd > $D/tl_alsd_$i.txt 2>&1
timeout 120 python scripts/timeline.py --algo greedy > $D/tl_greedy_$i.txt 2>&1
TBEAM_SEL_THREADS=256 timeout 120 python scripts/timeline.py --algo greedy > $D/tl_greedy256_$i.txt 2>&1
done
timeout 300 python scripts/gemm_trace.py 100 > $D/trace.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err

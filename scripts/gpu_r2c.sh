mkdir -p gpurun_out/r2c
D=gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -k "beam_32 or eos or merge_max or round_cap or max_len or wider or peaky or specialised or lstm" > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
for i in 1 2; do
timeout 120 python scripts/timeline.py --algo alsd > $D/tl_alsd_g12_$i.txt 2>&1
TBEAM_GATES8=1 timeout 120 python scripts/timeline.py --algo alsd > $D/tl_alsd_g8_$i.txt 2>&1
done
timeout 120 python scripts/timeline.py --algo greedy > $D/tl_greedy_g12.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err

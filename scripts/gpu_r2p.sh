mkdir -p gpurun_out/r2p
D=gpurun_out/r2p
export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -q --timeout 1200 -k "c3 or c4 or c5" > $D/pytest_cfg.log 2>&1; echo "rc=$?" >> $D/pytest_cfg.log
timeout 1200 python scripts/bench_configs.py --only c3,c4,c5 --reps 1 > $D/configs.jsonl 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err

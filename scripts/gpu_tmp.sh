mkdir -p gpurun_out/s3
D=gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
TBEAM_S3_PER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest_per1.log 2>&1; echo "rc=$?" >> $D/pytest_per1.log
export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_ref_adapter.py -q --timeout 800 -k "c1 or c2 or adapter" > $D/pytest_cfg.log 2>&1; echo "rc=$?" >> $D/pytest_cfg.log
timeout 600 python scripts/bench_configs.py --only c1,c2 --reps 2 > $D/configs.jsonl 2>&1
TBEAM_FP32_SIMT=1 timeout 600 python scripts/bench_configs.py --only c2 --reps 2 > $D/configs_simt.jsonl 2>&1

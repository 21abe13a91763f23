mkdir -p gpurun_out/s3b
D=gpurun_out/s3b
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
TBEAM_S3_PER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest_per1.log 2>&1; echo "rc=$?" >> $D/pytest_per1.log
rm -f $D/parity_log.jsonl; export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_ref_adapter.py -q --timeout 800 -k "c1 or c2 or adapter" > $D/pytest_cfg.log 2>&1; echo "rc=$?" >> $D/pytest_cfg.log
timeout 600 python scripts/bench_configs.py --only c1,c2 --reps 2 > $D/configs.jsonl 2>&1
timeout 300 python scripts/timeline.py --config c2 --precision fp32 --algo aes --frames 200 > $D/timeline.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c2 > $D/trace.txt 2>&1
TBEAM_S3_CLUSTER=0 timeout 600 python scripts/bench_configs.py --only c2 --reps 2 > $D/configs_noclu.jsonl 2>&1

mkdir -p gpurun_out/r2h
D=gpurun_out/r2h
export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -k cluster > $D/pytest_cluster.log 2>&1; echo "rc=$?" >> $D/pytest_cluster.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -rf --timeout 900 -k "c4 or c5" > $D/pytest_cfg.log 2>&1; echo "rc=$?" >> $D/pytest_cfg.log
timeout 900 python scripts/bench_configs.py --only c4,c5 --reps 1 > $D/configs.jsonl 2> $D/configs.err
TBEAM_JOINT_CLUSTER=0 timeout 900 python scripts/bench_configs.py --only c4,c5 --reps 1 > $D/configs_nocl.jsonl 2> $D/configs_nocl.err

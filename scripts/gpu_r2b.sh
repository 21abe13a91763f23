mkdir -p gpurun_out/r2b
D=gpurun_out/r2b
export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
timeout 300 python scripts/bench_configs.py --only c1,c2 > $D/c12.jsonl 2>&1
TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_acc32.so timeout 300 python scripts/bench_configs.py --only c2 > $D/c2_acc32.jsonl 2>&1

mkdir -p gpurun_out/mg
D=gpurun_out/mg
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 1500 python -m pytest tests/test_gpu_configs.py -q --timeout 1200 -k "c5" > $D/pytest_cfg.log 2>&1; echo "rc=$?" >> $D/pytest_cfg.log
unset TBEAM_PARITY_LOG
for v in base lists; do
  if [ $v = base ]; then L=$PWD/paper_2506_00185_b200/libtbeam_b200.so; else L=$PWD/paper_2506_00185_b200/variants/libtbeam_$v.so; fi
  TBEAM_LIB=$L timeout 600 python scripts/gemm_trace.py 40 c5 > $D/trace_$v.txt 2>&1
  TBEAM_LIB=$L timeout 900 python scripts/bench_configs.py --only c5 --reps 1 > $D/c5_$v.jsonl 2>&1
done

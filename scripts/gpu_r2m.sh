mkdir -p gpurun_out/r2m
D=gpurun_out/r2m
for v in 0 1; do
  if [ $v = 0 ]; then unset TBEAM_NO_FK; else export TBEAM_NO_FK=1; fi
  timeout 900 python scripts/bench_configs.py --only c3,c4 --reps 2 > $D/configs_nofk$v.jsonl 2>&1
  timeout 300 python scripts/timeline.py --config c3 --algo aes --frames 100 > $D/tl_c3_nofk$v.txt 2>&1
  timeout 120 python scripts/timeline.py --algo alsd > $D/tl_bench_nofk$v.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x --timeout 900 -k "c3 or c4 or bench" > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log

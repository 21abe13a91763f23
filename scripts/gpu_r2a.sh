mkdir -p gpurun_out/r2a
D=gpurun_out/r2a
export TBEAM_PARITY_LOG=$D/parity_log.jsonl
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 900 > $D/pytest.log 2>&1; echo "rc=$?" >> $D/pytest.log
for v in acc64 exactexp acc64exp; do
  TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_$v.so timeout 300 python scripts/parity_configs.py --only c2 > $D/c2_$v.jsonl 2>&1
done
timeout 400 python bench.py --steps 5 --warmup 3 > $D/bench.json 2> $D/bench.err
TBEAM_DIST_BACKEND=gloo timeout 400 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $D/bench_g2.json 2> $D/bench_g2.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err

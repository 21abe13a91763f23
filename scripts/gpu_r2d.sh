mkdir -p gpurun_out/r2d
D=gpurun_out/r2d
for v in accchunk acc32; do
  TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_$v.so timeout 300 python scripts/parity_configs.py --only c2,c1 > $D/par_$v.jsonl 2>&1
  TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_$v.so timeout 300 python scripts/bench_configs.py --only c2 > $D/c2_$v.jsonl 2>&1
done
timeout 300 python scripts/bench_configs.py --only c2 > $D/c2_acc64.jsonl 2>&1

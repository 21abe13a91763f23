mkdir -p gpurun_out/r2e
D=gpurun_out/r2e
for v in fold8 fold16; do
  TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_$v.so timeout 300 python scripts/parity_configs.py --only c2 > $D/par_$v.jsonl 2>&1
  TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_$v.so timeout 300 python scripts/bench_configs.py --only c2 > $D/c2_$v.jsonl 2>&1
done

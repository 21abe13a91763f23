mkdir -p gpurun_out/ab4
D=gpurun_out/ab4
TBEAM_LIB=$PWD/paper_2506_00185_b200/variants/libtbeam_ab5.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $D/pytest_ab5.log 2>&1; echo "rc=$?" >> $D/pytest_ab5.log
for pass in 1 2; do
for v in base ab5 ab1; do
  if [ $v = base ]; then L=$PWD/paper_2506_00185_b200/libtbeam_b200.so; else L=$PWD/paper_2506_00185_b200/variants/libtbeam_$v.so; fi
  for a in alsd greedy; do
    echo "== $v $a pass $pass" >> $D/ab.txt
    TBEAM_LIB=$L timeout 300 python scripts/timeline.py --algo $a 2>&1 | grep -E "decode|busy" >> $D/ab.txt
  done
  TBEAM_LIB=$L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_${v}_$pass.json 2>/dev/null
done
done

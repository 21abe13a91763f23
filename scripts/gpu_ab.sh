# A/B of measurement variants (paper_2506_00185_b200/variants/*.so) against the
# in-tree library: round timeline of the bench workload per variant, 2 passes
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/ab
ALGOS=${ALGOS:-alsd}
for pass in 1 2; do
  for v in base $(ls paper_2506_00185_b200/variants/ 2>/dev/null | sed 's/libtbeam_//; s/\.so//'); do
    for a in $ALGOS; do
      if [ $v = base ]; then L=paper_2506_00185_b200/libtbeam_b200.so; else L=paper_2506_00185_b200/variants/libtbeam_$v.so; fi
      echo "== $v $a pass $pass" >> gpurun_out/ab/ab.txt
      TBEAM_LIB=$PWD/$L timeout 300 python scripts/timeline.py --algo $a $TLARGS 2>&1 | head -6 >> gpurun_out/ab/ab.txt
    done
  done
done
cat gpurun_out/ab/ab.txt

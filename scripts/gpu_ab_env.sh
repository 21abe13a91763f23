# timelines of the bench workload and C3/C4 (+ select phase traces) for the
# in-tree library, with the env overrides given in $ENVS (space-separated
# groups joined by ';'), e.g. ENVS="X=1;TBEAM_SEL_THREADS=128"
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/ab3; rm -f gpurun_out/ab3/ab.txt
IFS=';' read -ra GROUPS_ <<< "${ENVS:-X=1}"
for g in "${GROUPS_[@]}"; do
  for c in bench c3 c4; do
    echo "== $c $g" >> gpurun_out/ab3/ab.txt
    if [ $c = bench ]; then A="--algo alsd"; else A="--config $c --algo aes --frames 100"; fi
    env $g timeout 600 python scripts/timeline.py $A 2>&1 | head -6 >> gpurun_out/ab3/ab.txt
  done
done
for c in c3 c4; do timeout 600 python scripts/gemm_trace.py 100 $c > gpurun_out/ab3/trace_$c.txt 2>&1; done
cat gpurun_out/ab3/ab.txt gpurun_out/ab3/trace_c*.txt

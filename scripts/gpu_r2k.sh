mkdir -p gpurun_out/r2k
D=gpurun_out/r2k
for c in c3 c4; do
  timeout 300 python scripts/timeline.py --config $c --algo aes --frames 100 > $D/tl_${c}_aes.txt 2>&1
  timeout 300 python scripts/timeline.py --config $c --algo greedy --frames 100 > $D/tl_${c}_greedy.txt 2>&1
done
timeout 300 python scripts/timeline.py --config c3 --algo alsd --frames 100 > $D/tl_c3_alsd.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c3 > $D/trace_c3.txt 2>&1

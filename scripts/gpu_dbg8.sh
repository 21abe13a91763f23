mkdir -p gpurun_out/dbg8
for p in 0 1; do for a in 1 2; do
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python scripts/debug_k32.py $p $a > gpurun_out/dbg8/k32_${p}_${a}.txt 2>&1
done; done

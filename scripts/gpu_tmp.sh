mkdir -p gpurun_out/gr2
D=gpurun_out/gr2
for pass in 1 2; do
for r in 0 1; do
TBEAM_GATES_RING=$r timeout 1200 python scripts/bench_configs.py --only c3,c4 --reps 1 > $D/configs_r${r}_$pass.jsonl 2>&1
done
done

ALGOS="alsd greedy" bash scripts/gpu_ab.sh > /dev/null 2>&1
for pass in 1 2; do
 echo "== gates12 alsd pass $pass" >> gpurun_out/ab/ab.txt
 TBEAM_GATES12=1 timeout 300 python scripts/timeline.py --algo alsd 2>&1 | head -6 >> gpurun_out/ab/ab.txt
done
timeout 900 python scripts/bench_configs.py --only c3,c4 --reps 2 > gpurun_out/ab/configs.jsonl 2>&1

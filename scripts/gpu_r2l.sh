mkdir -p gpurun_out/r2l
D=gpurun_out/r2l
for bn in 0 64; do
  if [ $bn = 0 ]; then unset TBEAM_JOINT_BN; else export TBEAM_JOINT_BN=$bn; fi
  timeout 900 python scripts/bench_configs.py --only c3,c4 --reps 2 > $D/configs_bn$bn.jsonl 2>&1
  timeout 300 python scripts/timeline.py --config c3 --algo aes --frames 100 > $D/tl_c3_bn$bn.txt 2>&1
  timeout 120 python scripts/timeline.py --algo alsd > $D/tl_bench_bn$bn.txt 2>&1
done

mkdir -p gpurun_out/r2f
D=gpurun_out/r2f
for a in alsd greedy; do timeout 300 python scripts/concurrency_probe.py --algo $a --parts 2 > $D/conc_$a.txt 2>&1; done
timeout 300 python scripts/concurrency_probe.py --algo alsd --parts 4 > $D/conc_alsd4.txt 2>&1
TBEAM_SEL_THREADS=256 timeout 120 python scripts/timeline.py --algo alsd > $D/tl_sel256.txt 2>&1
timeout 120 python scripts/timeline.py --algo alsd > $D/tl_base.txt 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:^tc_gemm$ -s 3 -c 2 -o $D/c5_joint python scripts/profile_decode.py --reps 1 --graph 0 --config c5 --algo aes --frames 10 > $D/ncu_c5.log 2>&1
python scripts/ncu_summary.py $D/c5_joint.ncu-rep "C5 ring joint (tc_gemm<256, JointEpi<16,1>>)" > $D/c5_joint_summary.txt 2>&1
python scripts/ncu_traffic.py c5/bf16 $D/c5_joint.ncu-rep > $D/traffic_c5.log 2>&1
cp profiles/kernel_traffic.json $D/
rm -f $D/c5_joint.ncu-rep

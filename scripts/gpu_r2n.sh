mkdir -p gpurun_out/r2n
D=gpurun_out/r2n
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^tc_gemm$ -s 4 -c 1 -o $D/c5_joint python scripts/profile_decode.py --reps 1 --graph 0 --config c5 --algo aes --frames 8 > $D/ncu.log 2>&1
ncu -i $D/c5_joint.ncu-rep --page source --csv --print-source cuda,sass > $D/c5_joint_src.csv 2>/dev/null
python scripts/ncu_summary.py $D/c5_joint.ncu-rep "C5 joint" > $D/summary.txt 2>&1
rm -f $D/c5_joint.ncu-rep
gzip $D/c5_joint_src.csv

# ncu source-line profile of the C5 joint (tc_gemm<256, JointEpi<16, late>>)
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/ncu
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:JointEpi -s 6 -c 1 -o gpurun_out/ncu/joint_c5 python scripts/profile_decode.py --config c5 --algo aes --frames 12 --reps 1 --graph 0 > gpurun_out/ncu/joint_c5.log 2>&1
ncu -i gpurun_out/ncu/joint_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu/joint_c5.src.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/ncu/joint_c5.src.csv 50 > gpurun_out/ncu/joint_c5.lines.txt
ncu -i gpurun_out/ncu/joint_c5.ncu-rep --page details --csv > gpurun_out/ncu/joint_c5.details.csv 2>/dev/null
tail -2 gpurun_out/ncu/joint_c5.log

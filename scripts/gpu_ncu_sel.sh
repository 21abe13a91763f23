set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 60 -c 5 -o gpurun_out/prof_select python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu_full_select.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:JointEpi -s 60 -c 5 -o gpurun_out/prof_joint python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu_full_joint.log 2>&1
tail -3 gpurun_out/ncu_full_select.log gpurun_out/ncu_full_joint.log

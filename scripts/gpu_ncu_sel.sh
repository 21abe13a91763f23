# ncu source-line stall profile of the select kernel: bench workload and C3
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 40 -c 12 -o gpurun_out/ncu/sel_bench python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > gpurun_out/ncu/sel_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 40 -c 12 -o gpurun_out/ncu/sel_c3 python scripts/profile_decode.py --config c3 --algo aes --frames 40 --reps 1 --graph 0 > gpurun_out/ncu/sel_c3.log 2>&1
for f in sel_bench sel_c3; do ncu -i gpurun_out/ncu/$f.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu/$f.src.csv 2>/dev/null; python scripts/ncu_lines.py gpurun_out/ncu/$f.src.csv 40 > gpurun_out/ncu/$f.lines.txt; done
tail -2 gpurun_out/ncu/*.log; cat gpurun_out/ncu/*.lines.txt

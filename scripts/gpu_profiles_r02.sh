# round-2 measurement pass for profiles/r02: launch list + ncu --set full of
# the per-round kernels (bench, C4 late-LM, C5 ring joint), DRAM traffic json
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
A=gpurun_out/prof2; mkdir -p $A
PD="python scripts/profile_decode.py --reps 1 --graph 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_alsd_T40.csv $PD --frames 40 > $A/ncu_launch.log 2>&1
python scripts/launch_summary.py $A/launches_alsd_T40.csv > $A/launches_alsd_T40.summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_greedy_T40.csv $PD --frames 40 --algo greedy > $A/ncu_launch_g.log 2>&1
python scripts/launch_summary.py $A/launches_greedy_T40.csv > $A/launches_greedy_T40.summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_fk -s 60 -c 6 -o $A/bench_fk $PD --frames 40 > $A/ncu_bench_fk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 30 -c 3 -o $A/bench_select $PD --frames 40 > $A/ncu_bench_select.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"tc_gemm|select_kernel" -s 40 -c 6 -o $A/c4 $PD --config c4 --algo aes --frames 30 > $A/ncu_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"tc_gemm<|select_kernel" -s 6 -c 4 -o $A/c5 $PD --config c5 --algo aes --frames 10 > $A/ncu_c5.log 2>&1
python scripts/ncu_traffic.py bench/bf16 $A/bench_fk.ncu-rep $A/bench_select.ncu-rep > $A/traffic.log 2>&1
python scripts/ncu_traffic.py c4/bf16 $A/c4.ncu-rep >> $A/traffic.log 2>&1
python scripts/ncu_traffic.py c5/bf16 $A/c5.ncu-rep >> $A/traffic.log 2>&1
cp profiles/kernel_traffic.json $A/kernel_traffic.json
{ python scripts/ncu_summary.py $A/bench_fk.ncu-rep "full-K GEMMs (joint / gates / proj), bench shape T=40";
  python scripts/ncu_summary.py $A/bench_select.ncu-rep "select kernel, bench shape T=40";
  python scripts/ncu_summary.py $A/c4.ncu-rep "C4 (AES++ K=8, 4-gram LM late + scored blank): joint + select";
  python scripts/ncu_summary.py $A/c5.ncu-rep "C5 (TDT AES++ K=16, V=8192, LM): ring joint + select"; } > $A/ncu_full_summary.txt 2>&1
rm -f $A/c5.ncu-rep $A/c4.ncu-rep
for a in alsd aes greedy; do timeout 300 python scripts/timeline.py --algo $a > $A/timeline_$a.txt 2>&1; done
timeout 300 python scripts/gemm_trace.py 100 > $A/trace_bench.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $A/bench.json 2> $A/bench.err

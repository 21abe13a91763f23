# round-2 final measurement pass: launch lists + ncu --set full of the bench
# per-round kernels (full-K GEMMs with two A boxes, select) and of the fp32
# tensor-core GEMMs (C2, tc_gemm_s3), DRAM traffic json, timelines, and
# compute-sanitizer memcheck of the fp32 tensor-core modes
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
A=gpurun_out/prof3; mkdir -p $A
PD="python scripts/profile_decode.py --reps 1 --graph 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_alsd_T40.csv $PD --frames 40 > $A/ncu_launch.log 2>&1
python scripts/launch_summary.py $A/launches_alsd_T40.csv > $A/launches_alsd_T40.summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_greedy_T40.csv $PD --frames 40 --algo greedy > $A/ncu_launch_g.log 2>&1
python scripts/launch_summary.py $A/launches_greedy_T40.csv > $A/launches_greedy_T40.summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_c2_T40.csv $PD --config c2 --precision fp32 --algo aes --frames 40 > $A/ncu_launch_c2.log 2>&1
python scripts/launch_summary.py $A/launches_c2_T40.csv > $A/launches_c2_T40.summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_fk -s 60 -c 6 -o $A/bench_fk $PD --frames 40 > $A/ncu_bench_fk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 30 -c 3 -o $A/bench_select $PD --frames 40 > $A/ncu_bench_select.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_s3 -s 30 -c 6 -o $A/c2_s3 $PD --config c2 --precision fp32 --algo aes --frames 40 > $A/ncu_c2_s3.log 2>&1
python scripts/ncu_traffic.py bench/bf16 $A/bench_fk.ncu-rep $A/bench_select.ncu-rep > $A/traffic.log 2>&1
python scripts/ncu_traffic.py c2/fp32 $A/c2_s3.ncu-rep >> $A/traffic.log 2>&1
cp profiles/kernel_traffic.json $A/kernel_traffic.json
{ python scripts/ncu_summary.py $A/bench_fk.ncu-rep "full-K GEMMs (joint / gates / proj), bench shape T=40";
  python scripts/ncu_summary.py $A/bench_select.ncu-rep "select kernel, bench shape T=40";
  python scripts/ncu_summary.py $A/c2_s3.ncu-rep "fp32 tensor-core GEMMs tc_gemm_s3 (C2: AES++ K=4, LSTM, fp32), T=40"; } > $A/ncu_full_summary.txt 2>&1
for a in alsd aes greedy; do timeout 300 python scripts/timeline.py --algo $a > $A/timeline_$a.txt 2>&1; done
timeout 300 python scripts/timeline.py --config c2 --precision fp32 --algo aes --frames 200 > $A/timeline_c2.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 > $A/trace_bench.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c2 > $A/trace_c2.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32_tensor_core_modes or gates_ring" > $A/memcheck_fp32_tc.log 2>&1; echo "rc=$?" >> $A/memcheck_fp32_tc.log
rm -f $A/*.ncu-rep
tail -3 $A/memcheck_fp32_tc.log

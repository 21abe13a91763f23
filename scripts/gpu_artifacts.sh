# full measurement pass for profiles/: parity, smoke, bench (+ reference arm),
# every BASELINE config, launch timelines, phase traces, ncu launch list and
# ncu --set full summaries of the per-round kernels
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
A=gpurun_out/art; mkdir -p $A
timeout 900 python -m pytest tests -m gpu -q > $A/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $A/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $A/smoke.log 2>&1; echo "smoke rc=$?" >> $A/smoke.log
timeout 900 python bench.py > $A/bench.json 2> $A/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $A/bench_reference.json 2>&1
for a in alsd aes greedy; do timeout 300 python scripts/timeline.py --algo $a > $A/timeline_$a.txt 2>&1; done
for c in c3 c4; do timeout 600 python scripts/timeline.py --config $c --algo aes --frames 100 > $A/timeline_$c.txt 2>&1; done
timeout 900 python scripts/timeline.py --config c5 --algo aes --frames 60 > $A/timeline_c5.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 > $A/trace_bench.txt 2>&1
timeout 300 python scripts/gemm_trace.py 100 c3 > $A/trace_c3.txt 2>&1
timeout 600 python scripts/gemm_trace.py 40 c5 > $A/trace_c5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $A/launches_alsd_T40.csv python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > $A/ncu_launch.log 2>&1
python scripts/launch_summary.py $A/launches_alsd_T40.csv > $A/launches_alsd_T40.summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_fk -s 60 -c 6 -o $A/prof_fk python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > $A/ncu_full_fk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 30 -c 3 -o $A/prof_select python scripts/profile_decode.py --frames 40 --reps 1 --graph 0 > $A/ncu_full_select.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:^tc_gemm$ -s 3 -c 2 -o $A/prof_c5_joint python scripts/profile_decode.py --config c5 --algo aes --frames 12 --reps 1 --graph 0 > $A/ncu_full_c5.log 2>&1
{ python scripts/ncu_summary.py $A/prof_fk.ncu-rep "full-K GEMMs (joint / gates / proj), bench shape T=40";
  python scripts/ncu_summary.py $A/prof_select.ncu-rep "select kernel, bench shape T=40";
  python scripts/ncu_summary.py $A/prof_c5_joint.ncu-rep "C5 joint (ring GEMM, BN=256, K=16 + LM), T=12"; } > $A/ncu_full_summary.txt 2>&1
timeout 1500 python scripts/bench_configs.py --only c1,c2,c3,c4 > $A/configs_c1_c4.jsonl 2> $A/configs_c1_c4.err
timeout 2000 python scripts/bench_configs.py --only c5 --reps 1 > $A/configs_c5.jsonl 2> $A/configs_c5.err
rm -f $A/prof_c5_joint.ncu-rep  # (summary kept; the report would crowd the 64 MiB copy-back)
tail -1 $A/pytest_gpu.log; cat $A/smoke.log; cat $A/launches_alsd_T40.summary.txt; head -c 400 $A/bench.json; echo; cat $A/configs_c1_c4.jsonl $A/configs_c5.jsonl | cut -c1-200; tail -n 3 $A/*.err

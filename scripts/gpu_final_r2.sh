# round-2 checkpoint: full GPU parity suite, smoke, bench (+ reference arm),
# every BASELINE config, C5 strong-scaling bench mode, timelines
set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
A=gpurun_out/final2; mkdir -p $A
export TBEAM_PARITY_LOG=$A/parity_log.jsonl
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 1200 > $A/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $A/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $A/smoke.log 2>&1; echo "smoke rc=$?" >> $A/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $A/bench.json 2> $A/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $A/bench_reference.json 2> $A/bench_reference.err
timeout 2400 python scripts/bench_configs.py > $A/configs.jsonl 2> $A/configs.err
timeout 1200 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline > $A/bench_c5.json 2> $A/bench_c5.err
for a in alsd aes greedy; do timeout 300 python scripts/timeline.py --algo $a > $A/timeline_$a.txt 2>&1; done
tail -1 $A/pytest_gpu.log; tail -1 $A/smoke.log

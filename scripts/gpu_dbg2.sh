mkdir -p gpurun_out/dbg2
D=gpurun_out/dbg2
P="python scripts/debug_parity.py --config c5 --streams 205,614"
timeout 300 $P --len 40 > $D/len40.jsonl 2>&1
timeout 300 $P --len 200 > $D/len200.jsonl 2>&1
timeout 300 $P --blank omit > $D/omit.jsonl 2>&1
timeout 300 $P --prune early > $D/early.jsonl 2>&1
timeout 300 $P --beam 12 > $D/k12.jsonl 2>&1
timeout 300 $P --merge max > $D/max.jsonl 2>&1
TBEAM_FORCE_SIMT=1 timeout 600 $P > $D/simt.jsonl 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scripts/debug_parity.py --config c5 --streams 205 --beam 8 --len 12 > $D/k8_memcheck.txt 2>&1

mkdir -p gpurun_out/dbg3
D=gpurun_out/dbg3
timeout 300 python scripts/round_diff.py --config c5 --stream 205 --len 40 > $D/rd_c5_205.txt 2>&1
timeout 300 python scripts/round_diff.py --config c3 --stream 8 --algo aes > $D/rd_c3_8.txt 2>&1
timeout 300 python scripts/round_diff.py --config c3 --stream 59 --algo aes > $D/rd_c3_59.txt 2>&1
P="python scripts/debug_parity.py --config c5 --streams 205,614"
timeout 300 $P --beam 8 > $D/k8.jsonl 2>&1
timeout 300 $P --beam 12 > $D/k12.jsonl 2>&1
TBEAM_FORCE_SIMT=1 timeout 600 $P --len 300 > $D/simt.jsonl 2>&1

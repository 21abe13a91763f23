mkdir -p gpurun_out/dbg6
D=gpurun_out/dbg6
timeout 300 python scripts/round_diff.py --config c5 --stream 614 --len 80 --tol 3e-3 > $D/rd_614.txt 2>&1
TBEAM_SEL_GENERIC=16 timeout 300 python scripts/debug_parity.py --config c5 --streams 205,614 --len 300 > $D/generic16.jsonl 2>&1

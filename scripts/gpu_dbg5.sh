mkdir -p gpurun_out/dbg5
D=gpurun_out/dbg5
timeout 300 python scripts/round_diff.py --config c5 --stream 614 --len 300 --tol 3e-3 > $D/rd_614.txt 2>&1
timeout 300 python scripts/round_diff.py --config c5 --stream 205 --len 300 --tol 3e-3 > $D/rd_205.txt 2>&1

mkdir -p gpurun_out/dbg7
TBEAM_LIB=paper_2506_00185_b200/variants/libtbeam_dbgpfx.so ORACLE_DEBUG_T=52 timeout 300 python scripts/round_diff.py --config c5 --stream 614 --len 60 --tol 3e-3 > gpurun_out/dbg7/rd.txt 2>&1

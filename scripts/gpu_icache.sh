timeout 300 python scripts/timeline.py --algo greedy > gpurun_out/tl_base.txt 2>&1
TBEAM_LIB=$PWD/paper_2506_00185_b200/libtbeam_pad.so timeout 300 python scripts/timeline.py --algo greedy > gpurun_out/tl_pad.txt 2>&1
cat gpurun_out/tl_base.txt gpurun_out/tl_pad.txt

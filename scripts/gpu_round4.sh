timeout 600 python scripts/timeline.py --config c5 --algo aes --frames 60 > gpurun_out/timeline_c5.txt 2>&1
timeout 600 python scripts/timeline.py --config c5 --algo greedy --frames 60 > gpurun_out/timeline_c5_greedy.txt 2>&1
timeout 600 python scripts/timeline.py --config c3 --algo alsd --frames 100 > gpurun_out/timeline_c3.txt 2>&1
cat gpurun_out/timeline_c5.txt gpurun_out/timeline_c5_greedy.txt gpurun_out/timeline_c3.txt

mkdir -p gpurun_out/r2base
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r2base/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2base/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2base/bench.json 2> gpurun_out/r2base/bench.err
timeout 120 python scripts/timeline.py --algo alsd > gpurun_out/r2base/tl_alsd.txt 2>&1
timeout 120 python scripts/timeline.py --algo greedy > gpurun_out/r2base/tl_greedy.txt 2>&1
nproc > gpurun_out/r2base/nproc.txt

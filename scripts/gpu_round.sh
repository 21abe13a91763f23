set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_fp32.log 2>&1
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench_fp32.log; tail -c 3000 gpurun_out/bench_bf16.log; tail -c 1500 gpurun_out/bench_ref.log

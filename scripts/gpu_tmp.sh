mkdir -p gpurun_out/r2u
for k in 2 4 8; do TBEAM_SPLITK=$k timeout 600 python scripts/bench_configs.py --only c1,c2 > gpurun_out/r2u/configs_sk$k.jsonl 2>&1; done

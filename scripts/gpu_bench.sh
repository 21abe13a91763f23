set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 5000 gpurun_out/bench.json

set -e; test -f paper_2506_00185_b200/libtbeam_b200.so || { echo "NO LIBRARY"; exit 1; }; set +e
for v in b200 A B; do TBEAM_LIB=$PWD/paper_2506_00185_b200/libtbeam_$v.so timeout 300 python scripts/timeline.py --algo alsd > gpurun_out/tl_$v.txt 2>&1; echo "== $v"; head -6 gpurun_out/tl_$v.txt; done

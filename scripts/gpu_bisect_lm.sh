echo "== HEAD lib"; TBEAM_LIB=$PWD/paper_2506_00185_b200/libtbeam_head.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lm_fusion_tensor_core" 2>&1 | tail -n 12 | cut -c1-200
echo "== new lib"; timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lm_fusion_tensor_core" 2>&1 | tail -n 12 | cut -c1-200

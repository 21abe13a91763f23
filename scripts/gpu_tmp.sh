mkdir -p gpurun_out/s3t
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "fp32_tensor_core_modes" > gpurun_out/s3t/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3t/pytest.log

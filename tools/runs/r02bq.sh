set -u
mkdir -p gpurun_out
T=r02bq
timeout 600 python -m pytest tests/test_fp8_gpu.py -x -q -k "zero_blocks" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"

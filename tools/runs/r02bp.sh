set -u
mkdir -p gpurun_out
T=r02bp
timeout 600 python -m pytest tests/test_fp8_gpu.py -x -q -k "negative_alpha" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"

set -u
mkdir -p gpurun_out
T=r02br
timeout 600 python -m pytest tests/test_bwd_gpu.py -x -q -k "matches_oracle" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"

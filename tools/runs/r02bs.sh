set -u
mkdir -p gpurun_out
T=r02bs
timeout 600 python -m pytest tests/test_fwd_gpu.py -x -q -k "tiny_and_ragged" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"

set -u
mkdir -p gpurun_out
T=r02ba
timeout 900 python -m pytest tests/test_fwd_gpu.py -x -q -k "aligned or strided" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/prep_time.py > gpurun_out/${T}_prep.log 2>&1; echo "prep rc=$?"

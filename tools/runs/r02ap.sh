set -u
mkdir -p gpurun_out
T=r02ap
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" > gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep rc=$?"
for i in 1 2; do
FA3B_K5_TMA=0 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "direct rc=$?"
FA3B_K5_TMA=1 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "tma rc=$?"
done
timeout 600 python -m pytest tests/test_fp8_gpu.py -x -q > gpurun_out/${T}_pytest_fp8.log 2>&1; echo "pytest fp8 rc=$?"

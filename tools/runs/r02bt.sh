set -u
mkdir -p gpurun_out
T=r02bt
FA3B_K5_GROUPS=3 timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" > gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep groups rc=$?"
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" >> gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep rc=$?"
for i in 1 2; do
FA3B_K5_GROUPS=1 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "g1 rc=$?"
FA3B_K5_GROUPS=3 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "g3 rc=$?"
done

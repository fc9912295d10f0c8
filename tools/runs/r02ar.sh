set -u
mkdir -p gpurun_out
T=r02ar
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" > gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep rc=$?"
FA3B_K5_LPR=1 timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" >> gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep lpr1 rc=$?"
for i in 1 2; do
FA3B_K5_LPR=1 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "lpr1 rc=$?"
FA3B_K5_LPR=2 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "lpr2 rc=$?"
done
bash tools/ncu_prep.sh ${T}_k5_lpr2

set -u
mkdir -p gpurun_out
T=r02aq
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" > gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep rc=$?"
for i in 1 2; do
FA3B_K5_ROW=0 FA3B_K5_TMA=0 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "direct rc=$?"
FA3B_K5_ROW=1 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "row rc=$?"
done
PREP_DATA=narrow FA3B_K5_ROW=1 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "row narrow rc=$?"
bash tools/ncu_prep.sh ${T}_k5_row

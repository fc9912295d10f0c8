set -u
mkdir -p gpurun_out
T=r02ax
for L in 4 2; do FA3B_K5_LPR256=$L timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "prepare" >> gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep lpr256=$L rc=$?"; done
for i in 1 2; do for L in 0 2 4; do
FA3B_K5_LPR256=$L timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "lpr256=$L rc=$?"
done; done

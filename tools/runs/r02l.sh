set -u
mkdir -p gpurun_out
T=r02l
timeout 300 python tools/prep_time.py > gpurun_out/${T}_prep.log 2>&1
FA3B_K5_PF=0 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "prep rc=$?"
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k prepare > gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep rc=$?"
timeout 600 python tools/ab.py build/variants/spin.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"
bash tools/ncu_prep.sh ${T}_k5

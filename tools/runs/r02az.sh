set -u
mkdir -p gpurun_out
T=r02az
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q > gpurun_out/${T}_pytest_fp8.log 2>&1; echo "pytest fp8 rc=$?"
timeout 900 python tools/ab.py build/variants/base2.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_pack_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/base2.so >> gpurun_out/${T}_pack_ab.log 2>&1; echo "ab2 rc=$?"
FA3B_LIB=build/variants/base2.so timeout 300 python tools/prep_time.py > gpurun_out/${T}_prep.log 2>&1; echo "prep base rc=$?"
timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "prep new rc=$?"

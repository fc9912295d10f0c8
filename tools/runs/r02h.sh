set -u
mkdir -p gpurun_out
T=r02h
timeout 900 python -m pytest tests/test_fp8_gpu.py tests/test_report.py -x -q > gpurun_out/${T}_pytest_fp8.log 2>&1; echo "pytest fp8 rc=$?"
timeout 300 python tools/prep_time.py > gpurun_out/${T}_prep.log 2>&1; echo "prep rc=$?"
timeout 300 python tools/fp8_acc.py > gpurun_out/${T}_acc.log 2>&1
FA3B_FP8_THR=2 timeout 300 python tools/fp8_acc.py >> gpurun_out/${T}_acc.log 2>&1; echo "acc rc=$?"
timeout 600 python tools/ab.py build/variants/base.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"
FA3B_FP8_THR=2 timeout 600 python tools/ab.py build/variants/base.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_ab_thr2.log 2>&1; echo "ab2 rc=$?"
timeout 600 python -m pytest tests/test_fwd_gpu.py -x -q > gpurun_out/${T}_pytest_fwd.log 2>&1; echo "pytest fwd rc=$?"

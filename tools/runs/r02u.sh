set -u
mkdir -p gpurun_out
T=r02u
cat gpurun_out/r02t_mmaspin_ab.log 2>/dev/null | head -3
FA3B_FWD_P2=1 timeout 600 python -m pytest tests/test_fp8_gpu.py -x -q -k "error_band or many_items or beats" > gpurun_out/${T}_pytest_p2.log 2>&1; echo "pytest p2 rc=$?"
FA3B_FWD_P2=0 timeout 300 python tools/wide_ab.py > gpurun_out/${T}_p2_ab.log 2>&1
FA3B_FWD_P2=1 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_p2_ab.log 2>&1; echo "ab rc=$?"
FA3B_FWD_P2=1 timeout 300 python tools/fp8_acc.py > gpurun_out/${T}_acc.log 2>&1; echo "acc rc=$?"

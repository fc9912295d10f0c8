set -u
mkdir -p gpurun_out
T=r02f
timeout 600 python tools/ab.py build/variants/base.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"
for e in "FA3B_FP8_VHI=1" "FA3B_FP8_VHI=2" "FA3B_FP8_VHI=1 FA3B_FP8_THR=1" "FA3B_FP8_VHI=1 FA3B_FP8_THR=0" "FA3B_FP8_VHI=2 FA3B_FP8_THR=0"; do
  env $e timeout 300 python tools/fp8_acc.py >> gpurun_out/${T}_acc.log 2>&1
done
echo acc done
timeout 900 python -m pytest tests/test_fp8_gpu.py tests/test_report.py tests/test_fwd_gpu.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"

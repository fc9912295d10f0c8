set -u
mkdir -p gpurun_out
T=r02am
FA3B_LIB=build/variants/spec.so timeout 600 python -m pytest tests/test_fwd_gpu.py tests/test_fp8_gpu.py -x -q > gpurun_out/${T}_pytest_spec.log 2>&1; echo "pytest spec rc=$?"
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/spec.so > gpurun_out/${T}_spec_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py build/variants/spec.so paper_2407_08608_b200/libfa3b.so >> gpurun_out/${T}_spec_ab.log 2>&1; echo "ab2 rc=$?"

set -u
mkdir -p gpurun_out
T=r02au
timeout 900 python -m pytest tests/test_fwd_gpu.py tests/test_fp8_gpu.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/short_ab.py build/variants/base.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_v8_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/short_ab.py paper_2407_08608_b200/libfa3b.so build/variants/base.so >> gpurun_out/${T}_v8_ab.log 2>&1; echo "ab2 rc=$?"

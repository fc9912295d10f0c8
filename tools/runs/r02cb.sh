set -u
mkdir -p gpurun_out
T=r02cb
timeout 900 python -m pytest tests/test_fp8_gpu.py tests/test_fwd_gpu.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/ab.py build/variants/nochring8.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_chring8_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/nochring8.so >> gpurun_out/${T}_chring8_ab.log 2>&1; echo "ab2 rc=$?"
FA3B_LIB=build/variants/trace.so timeout 300 python tools/fwd_trace.py 256 > gpurun_out/${T}_trace_d256.log 2>&1; echo "trace rc=$?"

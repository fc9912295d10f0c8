set -u
mkdir -p gpurun_out
T=r02bn
timeout 900 python -m pytest tests/test_bwd_gpu.py tests/test_large_oracle_gpu.py -x -q > gpurun_out/${T}_pytest_bwd.log 2>&1; echo "pytest bwd rc=$?"
BWD_N=512,2048,8192 timeout 900 python tools/bwd_ab.py build/variants/dkts.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_dkss_ab.log 2>&1; echo "ab rc=$?"
BWD_N=512,2048,8192 timeout 900 python tools/bwd_ab.py paper_2407_08608_b200/libfa3b.so build/variants/dkts.so >> gpurun_out/${T}_dkss_ab.log 2>&1; echo "ab2 rc=$?"
FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_trace.py 128 > gpurun_out/${T}_bwd_trace.log 2>&1; echo "trace rc=$?"

set -u
mkdir -p gpurun_out
T=r02bc
timeout 900 python -m pytest tests/test_bwd_gpu.py -x -q > gpurun_out/${T}_pytest_bwd.log 2>&1; echo "pytest bwd rc=$?"
BWD_N=512,1024,2048,8192 timeout 900 python tools/bwd_ab.py build/variants/nokvpf.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_kvpf_ab.log 2>&1; echo "ab rc=$?"
BWD_N=512,1024,2048,8192 timeout 900 python tools/bwd_ab.py paper_2407_08608_b200/libfa3b.so build/variants/nokvpf.so >> gpurun_out/${T}_kvpf_ab.log 2>&1; echo "ab2 rc=$?"

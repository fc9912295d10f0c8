set -u
mkdir -p gpurun_out
T=r02bm
timeout 900 python -m pytest tests/test_bwd_gpu.py -x -q > gpurun_out/${T}_pytest_bwd.log 2>&1; echo "pytest bwd rc=$?"
BWD_N=1024,8192 timeout 900 python tools/bwd_ab.py build/variants/bsleep.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_spin_ab.log 2>&1; echo "ab rc=$?"
BWD_N=1024,8192 timeout 900 python tools/bwd_ab.py paper_2407_08608_b200/libfa3b.so build/variants/bsleep.so >> gpurun_out/${T}_spin_ab.log 2>&1; echo "ab2 rc=$?"

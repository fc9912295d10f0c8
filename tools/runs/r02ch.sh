set -u
mkdir -p gpurun_out
T=r02ch
timeout 900 python -m pytest tests/test_fwd_gpu.py -x -q > gpurun_out/${T}_pytest_fwd.log 2>&1; echo "pytest fwd rc=$?"
timeout 900 python tools/ab.py build/variants/chx0.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_chx_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/chx0.so >> gpurun_out/${T}_chx_ab.log 2>&1; echo "ab2 rc=$?"

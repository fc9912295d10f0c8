set -u
mkdir -p gpurun_out
T=r02m
timeout 600 python tools/ab.py build/variants/h2exp0.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"
timeout 300 python tools/fp8_acc.py > gpurun_out/${T}_acc.log 2>&1; echo "acc rc=$?"
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q > gpurun_out/${T}_pytest_fp8.log 2>&1; echo "pytest rc=$?"
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1

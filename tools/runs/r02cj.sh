set -u
mkdir -p gpurun_out
T=r02cj
timeout 900 python tools/ab.py build/variants/r02bo.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/r02bo.so >> gpurun_out/${T}_ab.log 2>&1; echo "ab2 rc=$?"

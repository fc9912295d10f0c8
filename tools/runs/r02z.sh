set -u
mkdir -p gpurun_out
T=r02z
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/thr3.so build/variants/thr4.so > gpurun_out/${T}_thr_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py build/variants/thr3.so paper_2407_08608_b200/libfa3b.so build/variants/thr4.so >> gpurun_out/${T}_thr_ab.log 2>&1; echo "ab rc=$?"

set -u
mkdir -p gpurun_out
T=r02cl
BWD_N=2048,8192 timeout 900 python tools/bwd_ab.py paper_2407_08608_b200/libfa3b.so build/variants/bemu3.so build/variants/bemu4.so > gpurun_out/${T}_bemu_ab.log 2>&1; echo "ab rc=$?"
BWD_N=2048,8192 timeout 900 python tools/bwd_ab.py build/variants/bemu4.so build/variants/bemu3.so paper_2407_08608_b200/libfa3b.so >> gpurun_out/${T}_bemu_ab.log 2>&1; echo "ab2 rc=$?"

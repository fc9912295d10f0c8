set -u
mkdir -p gpurun_out
T=r02ad
timeout 900 python tools/short_ab.py build/variants/noqpf.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_qprefetch_ab.log 2>&1; echo "ab rc=$?"

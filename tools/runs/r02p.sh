set -u
mkdir -p gpurun_out
T=r02p
timeout 600 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/regs104.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"

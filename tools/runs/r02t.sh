set -u
mkdir -p gpurun_out
T=r02t
timeout 600 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/mmaspin.so > gpurun_out/${T}_mmaspin_ab.log 2>&1; echo "ab rc=$?"

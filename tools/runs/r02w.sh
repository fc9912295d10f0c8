set -u
mkdir -p gpurun_out
T=r02w
timeout 900 python tools/ab.py build/variants/prev.so paper_2407_08608_b200/libfa3b.so build/variants/nowd.so build/variants/spin2.so > gpurun_out/${T}_wait_ab.log 2>&1; echo "ab rc=$?"

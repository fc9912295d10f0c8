set -u
mkdir -p gpurun_out
T=r02bw
timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/thr5.so build/variants/thr6.so > gpurun_out/${T}_thr_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/ab.py build/variants/thr6.so build/variants/thr5.so paper_2407_08608_b200/libfa3b.so >> gpurun_out/${T}_thr_ab.log 2>&1; echo "ab2 rc=$?"

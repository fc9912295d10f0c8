set -u
mkdir -p gpurun_out
T=r02an
timeout 900 python tools/bwd_ab.py paper_2407_08608_b200/libfa3b.so build/variants/nosleep.so build/variants/b23d061.so build/variants/bac3b76.so > gpurun_out/${T}_bwd_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python tools/bwd_ab.py build/variants/bac3b76.so build/variants/b23d061.so build/variants/nosleep.so paper_2407_08608_b200/libfa3b.so >> gpurun_out/${T}_bwd_ab.log 2>&1; echo "ab2 rc=$?"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> gpurun_out/${T}_bwd_ab.log

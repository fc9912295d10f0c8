set -u
mkdir -p gpurun_out
T=r02ag
for n in 512 8192; do timeout 120 python tools/item_trace.py build/variants/trace.so $n > gpurun_out/${T}_items_n$n.log 2>&1; done
echo done

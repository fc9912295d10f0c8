set -u
mkdir -p gpurun_out
T=r02bg
for NN in 512 2048; do timeout 300 python tools/item_trace.py build/variants/trace.so $NN >> gpurun_out/${T}_items.log 2>&1; echo "items $NN rc=$?"; done

set -u
mkdir -p gpurun_out
T=r02bd
for NN in 512 8192; do FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_items.py $NN 128 >> gpurun_out/${T}_bwd_items.log 2>&1; echo "items $NN rc=$?"; done
FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_items.py 512 64 >> gpurun_out/${T}_bwd_items.log 2>&1; echo "items d64 rc=$?"

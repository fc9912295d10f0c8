set -u
mkdir -p gpurun_out
T=r02bb
for D in 64 128; do FA3B_LIB=build/variants/trace.so timeout 300 python tools/fwd_trace.py $D >> gpurun_out/${T}_trace.log 2>&1; echo "trace $D rc=$?"; done

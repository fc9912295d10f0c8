set -u
mkdir -p gpurun_out
T=r02bz
FA3B_LIB=build/variants/trace.so timeout 300 python tools/fwd_trace.py 256 > gpurun_out/${T}_trace_d256.log 2>&1; echo "trace rc=$?"

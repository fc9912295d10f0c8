set -u
mkdir -p gpurun_out
T=r02ce
FA3B_LIB=build/variants/trace.so timeout 300 python tools/fwd_trace.py 256 0 block > gpurun_out/${T}_trace_fp8_d256.log 2>&1; echo "trace rc=$?"
FA3B_LIB=build/variants/trace.so timeout 300 python tools/fwd_trace.py 128 0 block > gpurun_out/${T}_trace_fp8_d128.log 2>&1; echo "trace rc=$?"

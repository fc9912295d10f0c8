set -u
mkdir -p gpurun_out
T=r02bl
FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_trace.py 128 > gpurun_out/${T}_bwd_trace.log 2>&1; echo "trace rc=$?"
FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_trace.py 64 >> gpurun_out/${T}_bwd_trace.log 2>&1; echo "trace64 rc=$?"

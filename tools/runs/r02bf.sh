set -u
mkdir -p gpurun_out
T=r02bf
timeout 900 python -m pytest tests/test_bwd_gpu.py tests/test_large_oracle_gpu.py -x -q > gpurun_out/${T}_pytest_bwd.log 2>&1; echo "pytest bwd rc=$?"
BWD_N=512,1024,2048,8192 timeout 900 python tools/bwd_ab.py build/variants/epig.so paper_2407_08608_b200/libfa3b.so build/variants/epikv2.so > gpurun_out/${T}_epi_ab.log 2>&1; echo "ab rc=$?"
BWD_N=512,1024,2048,8192 timeout 900 python tools/bwd_ab.py build/variants/epikv2.so paper_2407_08608_b200/libfa3b.so build/variants/epig.so >> gpurun_out/${T}_epi_ab.log 2>&1; echo "ab2 rc=$?"
for NN in 512; do FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_items.py $NN 128 >> gpurun_out/${T}_bwd_items.log 2>&1; FA3B_LIB=build/variants/trace.so timeout 300 python tools/bwd_items.py $NN 64 >> gpurun_out/${T}_bwd_items.log 2>&1; echo "items rc=$?"; done

set -u
mkdir -p gpurun_out
T=r02aj
timeout 900 python -m pytest tests/test_fp8_gpu.py tests/test_report.py -x -q > gpurun_out/${T}_pytest_fp8.log 2>&1; echo "pytest rc=$?"
FA3B_FWD_PAIRING=warp timeout 300 python tools/short_ab.py paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_short.log 2>&1
timeout 300 python tools/short_ab.py paper_2407_08608_b200/libfa3b.so >> gpurun_out/${T}_short.log 2>&1; echo "short rc=$?"

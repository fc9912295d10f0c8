set -u
mkdir -p gpurun_out
T=r02k
timeout 300 python tools/prep_time.py > gpurun_out/${T}_prep.log 2>&1
PREP_DATA=narrow timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "prep rc=$?"
timeout 600 python tools/ab.py build/variants/base.so paper_2407_08608_b200/libfa3b.so build/variants/emu1.so build/variants/emu3.so > gpurun_out/${T}_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k prepare > gpurun_out/${T}_pytest_prep.log 2>&1; echo "pytest prep rc=$?"
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
bash tools/ncu_fwd.sh ${T}_prof_bf16_d128c 128 1 0

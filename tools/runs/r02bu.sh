set -u
mkdir -p gpurun_out
T=r02bu
for i in 1 2 3; do
FA3B_LIB=build/variants/prevk5.so timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "prev rc=$?"
timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "cur rc=$?"
done

mkdir -p gpurun_out
for mode in "" "--torch"; do
REBK_HOST_TIMING=1 timeout 300 python tools/e2e_overhead.py c1 $mode > gpurun_out/e2e_c1.txt 2>&1; echo "mode=$mode rc=$?"
grep -v "^\[rebk host\]" gpurun_out/e2e_c1.txt | tail -4; grep "^\[rebk host\]" gpurun_out/e2e_c1.txt | tail -8
done

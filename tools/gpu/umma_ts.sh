mkdir -p gpurun_out
cd tools && timeout 60 ./umma_ts_test > ../gpurun_out/umma_ts.txt 2>&1; echo "rc=$?"; cat ../gpurun_out/umma_ts.txt

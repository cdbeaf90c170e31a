# ncu --set full of the C4 CSR kernel (300-iteration launch), after the plain run exits 0
B4="python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 300"
$B4 > gpurun_out/r02_c4_plain.json 2> gpurun_out/r02_c4_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:rebk_csr_kernel -c 1 -o gpurun_out/r02_c4_csr $B4 > gpurun_out/r02_c4_ncu.log 2>&1; echo c4_ncu_rc=$?
python tools/ncu_summary.py gpurun_out/r02_c4_csr.ncu-rep 300 > gpurun_out/r02_c4_csr_ncu.txt 2>&1; cat gpurun_out/r02_c4_csr_ncu.txt

# ncu --set full with source counters of the C5 persistent kernel (300-iteration launch); per-line stall samples as CSV
B5="python bench.py --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 300"
$B5 > gpurun_out/r02_c5_plain.json 2> gpurun_out/r02_c5_plain.err && \
ncu --set full --section SourceCounters --clock-control none --import-source on -k regex:k_rebk_mrhs_persistent -c 1 -o gpurun_out/r02_c5_pk_v2 $B5 > gpurun_out/r02_c5_ncu.log 2>&1; echo c5_ncu_rc=$?
python tools/ncu_summary.py gpurun_out/r02_c5_pk_v2.ncu-rep 300 > gpurun_out/r02_c5_pk_ncu_v2.txt 2>&1; cat gpurun_out/r02_c5_pk_ncu_v2.txt
ncu -i gpurun_out/r02_c5_pk_v2.ncu-rep --page source --csv > gpurun_out/r02_c5_pk_source.csv 2>/dev/null; wc -l gpurun_out/r02_c5_pk_source.csv; head -3 gpurun_out/r02_c5_pk_source.csv | cut -c1-600

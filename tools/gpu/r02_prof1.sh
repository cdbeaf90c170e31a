set -x
S='python -c "import __graft_entry__ as g; g.smoke()"'
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_ncu.log 2>&1; echo smoke_ncu_rc=$?
B3="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 40"
$B3 > gpurun_out/r02_c3_plain.json 2> gpurun_out/r02_c3_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:rebk_dense_stream -c 1 -o gpurun_out/r02_c3_stream $B3 > gpurun_out/r02_c3_ncu.log 2>&1; echo c3_ncu_rc=$?
B2="python bench.py --workload c2 --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 2000"
$B2 > gpurun_out/r02_c2_plain.json 2> gpurun_out/r02_c2_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:rebk_dense_split -c 1 -o gpurun_out/r02_c2_split $B2 > gpurun_out/r02_c2_ncu.log 2>&1; echo c2_ncu_rc=$?
B5="python bench.py --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 300"
$B5 > gpurun_out/r02_c5_plain.json 2> gpurun_out/r02_c5_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:k_rebk_mrhs_persistent -c 1 -o gpurun_out/r02_c5_pk $B5 > gpurun_out/r02_c5_ncu.log 2>&1; echo c5_ncu_rc=$?
ls -la gpurun_out/

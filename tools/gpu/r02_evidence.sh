# evidence refresh on the current tree: the reference's own suites through the device plugins, smoke + launch list,
# ncu full capture of the C3 stream kernel, virtual-rank timing of the sharded kernel
set -x
tools/run_reference_tests.sh run > gpurun_out/r02_reference_suite_via_shim.log 2>&1; tail -2 gpurun_out/r02_reference_suite_via_shim.log
(cd baseline/_ref/kaczmarz_tests && PYTHONPATH="$PWD/..:$GRAFT_REPO_ROOT" python -m pytest -q -p no:cacheprovider -p tools.ref_cli_plugin --rootdir . -c /dev/null test_cli.py) > gpurun_out/r02_reference_cli_via_plugin.log 2>&1; tail -2 gpurun_out/r02_reference_cli_via_plugin.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_ncu.log 2>&1; echo smoke_ncu_rc=$?
B3="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 40"
$B3 > gpurun_out/r02_c3_plain.json 2> gpurun_out/r02_c3_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:rebk_dense_stream -c 1 -o gpurun_out/r02_c3_stream_v2 $B3 > gpurun_out/r02_c3_ncu.log 2>&1; echo c3_ncu_rc=$?
python tools/ncu_summary.py gpurun_out/r02_c3_stream_v2.ncu-rep 40 > gpurun_out/r02_c3_stream_ncu_v2.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu"
$B > gpurun_out/r02_c3_launch_plain.json 2>/dev/null && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c3_launches.csv $B > gpurun_out/r02_c3_launches_ncu.log 2>&1; echo launches_rc=$?
python tools/shard_virtual_timing.py 2 > gpurun_out/r02_shard_virtual_timing_f.txt 2>&1; tail -12 gpurun_out/r02_shard_virtual_timing_f.txt

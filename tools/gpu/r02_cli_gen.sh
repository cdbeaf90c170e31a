# generators + CLI on the B200; the reference's own test_cli.py through this CLI; the reference suite via the shim
timeout 600 python -m pytest tests/test_generators.py tests/test_cli.py -q -p no:cacheprovider -m gpu 2>&1 | tail -5
cd baseline/_ref/kaczmarz_tests && PYTHONPATH="$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT" timeout 900 python -m pytest -q -p no:cacheprovider -p tools.ref_cli_plugin --rootdir . -c /dev/null test_cli.py 2>&1 | tail -8 > "$GRAFT_REPO_ROOT/gpurun_out/r02_ref_test_cli_via_device_cli.log"; cd "$GRAFT_REPO_ROOT"
cat gpurun_out/r02_ref_test_cli_via_device_cli.log
timeout 1200 tools/run_reference_tests.sh run > gpurun_out/r02_reference_suite_via_shim.log 2>&1; tail -5 gpurun_out/r02_reference_suite_via_shim.log

# C5 persistent kernel: GPU parity tests, bench, per-phase trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_rhs" > gpurun_out/c5_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c5_tests.log
timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/c5_bench.json'));print('c5 ms/solve', round(d['ms_per_step'],2), 'iters/s', round(d['value']), 'K', d['details']['K'], 'frac', round(d['roofline']['frac'],3))"
REBK_PK_TRACE=40 REBK_PK_TRACE_FILE=gpurun_out/pk_trace.bin timeout 300 python bench.py --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/c5_trace.err
python tools/pk_trace.py gpurun_out/pk_trace.bin 148

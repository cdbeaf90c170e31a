# C5: epilogue change check + bound experiments (no MMAs / no conversion / neither)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_rhs" > gpurun_out/c5_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c5_tests.log
for d in 0 32 64 96; do
REBK_PK_DBG=$d timeout 300 python bench.py --workload c5 --steps 2 --warmup 1 --max-iters 400 --no-e2e --no-cpu > gpurun_out/c5_dbg$d.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/c5_dbg$d.json'));print('dbg $d: us/iter', round(d['ms_per_step']*1e3/d['config']['K'],2))"
REBK_PK_DBG=$d REBK_PK_TRACE=40 REBK_PK_TRACE_FILE=gpurun_out/pk_trace.bin timeout 300 python bench.py --workload c5 --steps 1 --warmup 1 --max-iters 400 --no-e2e --no-cpu > /dev/null 2> /dev/null
python tools/pk_trace.py gpurun_out/pk_trace.bin 148 | head -12 | tail -11 | tr '\n' ' '; echo
done
timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_bench.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/c5_bench.json'));print('full solve ms', round(d['ms_per_step'],2), 'K', d['config']['K'])"

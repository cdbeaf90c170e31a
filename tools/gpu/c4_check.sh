mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sparse" > gpurun_out/c4_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c4_tests.log
REBK_PROF=1 timeout 300 python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu > gpurun_out/c4_bench.json 2> gpurun_out/c4_prof.err; echo "c4 rc=$?"
grep -A10 "rebk prof" gpurun_out/c4_prof.err | tail -11
timeout 300 python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu > gpurun_out/c4_bench.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/c4_bench.json'));print('c4', round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],2))"

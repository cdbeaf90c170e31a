# C5: grid-barrier fence variants (PK_GBAR_FENCE 2 default / 1 / 0)
mkdir -p gpurun_out
for v in default f1 f0; do
  if [ $v = default ]; then L=""; else L="REBK_LIB=$PWD/tools/librebk_$v.so"; fi
  env $L timeout 600 python -m pytest tests -m gpu -x -q -k "multi_rhs" > gpurun_out/c5_tests_$v.log 2>&1; echo "$v tests rc=$?"
  env $L timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_bench_$v.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5_bench_$v.json'));print('$v c5 ms/solve', round(d['ms_per_step'],2), 'K', d['config']['K'])"
done
REBK_LIB=$PWD/tools/librebk_f0.so REBK_PK_TRACE=40 REBK_PK_TRACE_FILE=gpurun_out/pk_trace.bin timeout 300 python bench.py --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2> gpurun_out/c5_trace.err
python tools/pk_trace.py gpurun_out/pk_trace.bin 148

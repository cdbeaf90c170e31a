mkdir -p gpurun_out
for v in default r3a4 r3a2; do
  if [ $v = default ]; then L=""; else L="REBK_LIB=$PWD/tools/librebk_$v.so"; fi
  env $L timeout 300 python bench.py --workload c5 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/c5r_$v.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5r_$v.json'));print('$v c5 ms/solve', round(d['ms_per_step'],2), 'K', d['config']['K'])"
  env $L REBK_PK_DBG=96 timeout 300 python bench.py --workload c5 --steps 2 --warmup 1 --max-iters 400 --no-e2e --no-cpu > gpurun_out/c5r_dbg.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5r_dbg.json'));print('   $v dbg96 us/iter', round(d['ms_per_step']*1e3/d['config']['K'],2))"
done

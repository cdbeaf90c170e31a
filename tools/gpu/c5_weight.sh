mkdir -p gpurun_out
for pass in 1 2; do
for v in default w6 w8; do
  if [ $v = default ]; then L=""; else L="REBK_LIB=$PWD/tools/librebk_$v.so"; fi
  env $L timeout 300 python bench.py --workload c5 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/c5w_$v.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5w_$v.json'));print('pass $pass $v c5 ms/solve', round(d['ms_per_step'],2), 'K', d['config']['K'])"
done
done

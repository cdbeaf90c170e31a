# C2 split kernel: row_progress update variants, A/B twice in alternating order
mkdir -p gpurun_out
for pass in 1 2; do
for v in default pe4 pc pe4c; do
  if [ $v = default ]; then L=""; else L="REBK_LIB=$PWD/tools/librebk_$v.so"; fi
  env $L timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sp_$v.json 2> /dev/null
  python -c "import json;d=json.load(open('gpurun_out/sp_$v.json'));print('pass $pass $v ms/solve', round(d['ms_per_step'],2), 'iters', d['config']['iters_per_solve'])"
done
done
for v in pe4c; do
REBK_LIB=$PWD/tools/librebk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "split or c2 or c1 or replay" > gpurun_out/sp_tests_$v.log 2>&1; echo "$v tests rc=$?"; tail -2 gpurun_out/sp_tests_$v.log
done

mkdir -p gpurun_out
for pass in 1 2; do
for ncc in 3 4 5 6; do
  REBK_SPLIT_NCC=$ncc timeout 120 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/sw.json 2> /dev/null
  echo "pass $pass ncc=$ncc $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],2))" 2>&1 | tail -1)"
done
done

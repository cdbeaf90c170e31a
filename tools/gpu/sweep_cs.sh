mkdir -p gpurun_out
for cs in 6 7 8; do
  REBK_CLUSTER=$cs timeout 120 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/sw.json 2> gpurun_out/sw.err
  echo "cs=$cs $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],2), d['config']['grid_ctas'], d['config']['kernel_path'])" 2>&1 | tail -1)"
done

# C2 split-kernel geometry sweep (cluster size, column-group clusters)
mkdir -p gpurun_out
for cs in 8 4 16 2; do
  for ncc in auto; do
    REBK_CLUSTER=$cs timeout 120 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/sw_cs${cs}.json 2> gpurun_out/sw_cs${cs}.err
    echo "cs=$cs rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sw_cs${cs}.json'));print(round(d['ms_per_step'],2), d['config']['grid_ctas'], d['config']['kernel_path'])" 2>&1 | tail -1)"
  done
done
for ncc in 3 4 5 6 7 8 9 10 11 12; do
  REBK_CLUSTER=4 REBK_SPLIT_NCC=$ncc timeout 120 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/sw.json 2> /dev/null
  echo "cs=4 ncc=$ncc $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],2), d['config']['grid_ctas'])" 2>&1 | tail -1)"
done

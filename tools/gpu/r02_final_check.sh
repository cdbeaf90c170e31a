# the driver's round-end sequence on the current tree: GPU tests, smoke, bench N=1 (ours + reference)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_final_ref.json 2> gpurun_out/r02_final_ref.err; echo "ref rc=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_final_ours.json 2> gpurun_out/r02_final_ours.err; echo "ours rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_final_torchrun1.json 2> gpurun_out/r02_final_torchrun1.err; echo "torchrun1 rc=$?"
for f in ref ours torchrun1; do python -c "import json; d=json.loads(open('gpurun_out/r02_final_$f.json').read().strip().splitlines()[-1]); print('$f', d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))"; done
# the driver's profiler pass over smoke(): every kernel must run under replay (rc 0)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke_ncu.log 2>&1; echo "ncu smoke rc=$?"
python tools/ncu_launch_summary.py gpurun_out/r02_final_smoke_launches.csv 2>/dev/null | head -20

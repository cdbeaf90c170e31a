mkdir -p gpurun_out; export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:shard --csv python bench.py --workload c3 --sharded --steps 1 --warmup 1 --max-iters 40 > gpurun_out/sh_ncu.csv 2> gpurun_out/sh_ncu.err; echo "ncu rc=$?"
python tools/ncu_launch_summary.py gpurun_out/sh_ncu.csv 2>&1 | head -20

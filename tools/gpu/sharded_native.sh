# native (C++ issue loop, NCCL via librebk) sharded path vs the Python loop, N=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded" > gpurun_out/sh_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sh_tests.log
timeout 900 python bench.py --workload c3 --sharded --steps 2 --warmup 1 > gpurun_out/bench_c3_sharded.json 2> gpurun_out/bench_c3_sharded.err; echo "native rc=$?"; tail -2 gpurun_out/bench_c3_sharded.err
python -c "import json;d=json.load(open('gpurun_out/bench_c3_sharded.json'));print('native', d['value'], d['ms_per_step'], d['config']['driver'])"
timeout 900 python bench.py --workload c3 --sharded --python-loop --steps 2 --warmup 1 > gpurun_out/bench_c3_sharded_py.json 2> /dev/null; echo "py rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_c3_sharded_py.json'));print('python', d['value'], d['ms_per_step'], d['config']['driver'])"

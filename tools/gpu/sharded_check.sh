# sharded path: GPU tests (virtual ranks + NCCL world size 1 chunked loop), C3 sharded bench at N=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded" > gpurun_out/sh_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sh_tests.log
timeout 900 python bench.py --workload c3 --sharded --steps 2 --warmup 1 > gpurun_out/bench_c3_sharded.json 2> gpurun_out/bench_c3_sharded.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_c3_sharded.err
cat gpurun_out/bench_c3_sharded.json

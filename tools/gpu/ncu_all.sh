# ncu --set full captures of the C5, C3 and C4 kernels (bounded iteration counts)
mkdir -p gpurun_out; export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none -k regex:persistent -c 1 -o gpurun_out/c5_pk_v3 python bench.py --workload c5 --steps 1 --warmup 1 --max-iters 300 --no-e2e --no-cpu > gpurun_out/ncu_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:stream_kernel -c 1 -o gpurun_out/c3_stream python bench.py --workload c3 --steps 1 --warmup 1 --max-iters 20 --no-e2e --no-cpu > gpurun_out/ncu_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:csr_kernel -c 1 -o gpurun_out/c4_csr python bench.py --workload c4 --steps 1 --warmup 1 --max-iters 300 --no-e2e --no-cpu > gpurun_out/ncu_c4.log 2>&1; echo "c4 rc=$?"

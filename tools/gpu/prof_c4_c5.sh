# C4 CSR kernel phase profile (REBK_PROF=1) + ncu --set full of the C5 persistent kernel (300 iterations)
mkdir -p gpurun_out; export PATH=/usr/local/cuda/bin:$PATH
REBK_PROF=1 timeout 300 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu > /dev/null 2> gpurun_out/c4_prof.err; echo "c4 prof rc=$?"; grep -A30 "rebk prof" gpurun_out/c4_prof.err | tail -32
timeout 900 ncu --set full --clock-control none -k regex:persistent -c 1 --import-source on -o gpurun_out/c5_pk_full python bench.py --workload c5 --steps 1 --warmup 1 --max-iters 300 --no-e2e --no-cpu > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"; tail -3 gpurun_out/ncu_c5.log

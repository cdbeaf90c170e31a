mkdir -p gpurun_out; export PATH=/usr/local/cuda/bin:$PATH
export REBK_LIB=$PWD/tools/librebk_sc8.so
timeout 200 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/sc8_bench.json 2>gpurun_out/sc8_bench.err; echo sc8 bench rc=$?
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:split -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 2000 > gpurun_out/ncu_c2_min.csv 2> gpurun_out/ncu_c2_min.err; echo ncu min rc=$?
timeout 900 ncu --set full --clock-control none -k regex:split -c 1 --import-source on -o gpurun_out/c2_split_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 2000 > gpurun_out/ncu_c2_full.log 2>&1; echo ncu full rc=$?
unset REBK_LIB
REBK_PK_TRACE=40 REBK_PK_TRACE_FILE=gpurun_out/pk_trace.bin timeout 300 python bench.py --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/c5_trace.json 2> gpurun_out/c5_trace.err; echo c5 trace rc=$?
python tools/pk_trace.py gpurun_out/pk_trace.bin 148 > gpurun_out/c5_trace.txt 2>&1

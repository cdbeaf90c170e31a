# DRAM bytes of the C3 streaming kernel (40 iterations) for the second-pass order / L2 hint variants
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --max-iters 40"
$B > /dev/null 2>&1 || exit 1
for v in "0 0" "1 0" "0 1" "1 1"; do set -- $v
  REBK_STREAM_REV=$1 REBK_STREAM_L2HINT=$2 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:rebk_dense_stream -c 1 --csv --log-file gpurun_out/r02_c3_dram_rev$1_hint$2.csv $B > /dev/null 2>&1
done

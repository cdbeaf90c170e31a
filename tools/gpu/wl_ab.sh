# A/B of librebk variants on a workload: usage: wl_ab.sh <workload> name1 name2 ... ("product" = the in-tree library)
wl=$1; shift
for pass in 1 2; do
for v in "$@"; do
  lib=$PWD/tools/librebk_$v.so; [ "$v" = product ] && lib=$PWD/paper_2001_04179_b200/librebk.so
  REBK_LIB=$lib timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$wl $v', round(d['ms_per_step'],3), 'ms/solve', round(d['value']), 'iters/s', d['details'].get('grid_ctas'), d['details'].get('kernel_path'))"
done
done

# A/B of librebk variants on C5: ms per solve (two passes each); usage: c5_ab.sh name1 name2 ...
for pass in 1 2; do
for v in "$@"; do
  REBK_LIB=$PWD/tools/librebk_$v.so timeout 300 python bench.py --workload c5 --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],2), 'ms/solve K', d['details']['K'])"
done
done

# every bench workload on one B200 (default steps), plus the reference arm for c2
mkdir -p gpurun_out
for w in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));r=d.get('roofline',{});e=d.get('e2e') or {};print('$w', round(d['value'],1), d['unit'], 'frac', r.get('frac'), 'e2e', e.get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_c2_ref.json 2> gpurun_out/bench_c2_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_c2_ref.json

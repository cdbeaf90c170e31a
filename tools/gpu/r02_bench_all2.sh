# every workload's bench line on the current tree, with each reference arm
for w in c1 c2 c4 c5; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r02_all_$w.json 2> gpurun_out/r02_all_$w.err; echo "$w rc=$?"; done
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_all_c3.json 2> gpurun_out/r02_all_c3.err; echo "c3 rc=$?"
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r02_all_c3_ref.json 2> gpurun_out/r02_all_c3_ref.err; echo "c3 ref rc=$?"
python bench.py --sharded --steps 5 --warmup 2 > gpurun_out/r02_all_c3_sharded_n1.json 2> gpurun_out/r02_all_c3_sharded_n1.err; echo "c3 sharded rc=$?"
for w in c1 c2 c4 c5; do python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/r02_all_${w}_ref.json 2> gpurun_out/r02_all_${w}_ref.err; echo "$w ref rc=$?"; done
python - <<'P'
import json
for w in ["c3","c3_sharded_n1","c2","c1","c4","c5"]:
    d=json.loads(open(f"gpurun_out/r02_all_{w}.json").read().strip().splitlines()[-1])
    r=None
    try: r=json.loads(open(f"gpurun_out/r02_all_{w}_ref.json").read().strip().splitlines()[-1])["value"]
    except Exception: pass
    print(w, round(d["value"],1), "frac", round(d["roofline"]["frac"],4), "e2e", round(d["e2e"]["value"],1), "ref", r, d["clocks"])
P

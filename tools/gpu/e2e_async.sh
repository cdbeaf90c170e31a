# async device upload during prepare(): GPU tests + C2 e2e A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for pass in 1 2; do
for v in 0 1; do
REBK_ASYNC_UPLOAD=$v timeout 400 python bench.py --no-cpu > gpurun_out/e2e_async$v.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/e2e_async$v.json'));print('async=$v value', round(d['value']), 'e2e', round(d['e2e']['value']), 'e2e ms/step', round(d['e2e']['time_to_tol_s']*1e3,1))"
done
done

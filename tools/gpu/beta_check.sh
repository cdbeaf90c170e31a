# device beta: GPU tests + timing against the host eigensolver (C1, C2)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_beta.py -x -q > gpurun_out/beta_tests.log 2>&1; echo "beta tests rc=$?"; tail -15 gpurun_out/beta_tests.log
timeout 600 python tools/beta_timing.py > gpurun_out/beta_timing.txt 2>&1; echo "timing rc=$?"; cat gpurun_out/beta_timing.txt

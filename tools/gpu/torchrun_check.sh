# the driver's multi-GPU launch form at N=1 (both arms)
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/tr_ours.json 2> gpurun_out/tr_ours.err; echo "ours rc=$?"; tail -c 600 gpurun_out/tr_ours.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/tr_ref.json 2> gpurun_out/tr_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/tr_ref.json

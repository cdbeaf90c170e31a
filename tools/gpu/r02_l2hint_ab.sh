# A/B of the L2 eviction hints on the C3 streaming kernel (single GPU + emulated ranks)
for h in 0 1 0 1; do echo "== REBK_STREAM_L2HINT=$h"; REBK_STREAM_L2HINT=$h python tools/shard_virtual_timing.py 3 2>&1 | head -2; done

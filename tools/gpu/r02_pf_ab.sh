# A/B of the L2 prefetch depth of the streaming kernel (C3, single GPU and 8 emulated ranks)
for pf in 0 2 4 8 4 0; do echo "== REBK_STREAM_PF=$pf"; REBK_STREAM_PF=$pf python tools/shard_virtual_timing.py 3 2>&1 | grep -E "single|8 emulated|1 emulated"; done

# A/B of the reversed second passes (C2, R2) and the L2 hints on the C3 streaming kernel
for v in "0 0" "1 0" "0 1" "1 1" "1 1"; do set -- $v; echo "== REBK_STREAM_REV=$1 REBK_STREAM_L2HINT=$2"; REBK_STREAM_REV=$1 REBK_STREAM_L2HINT=$2 python tools/shard_virtual_timing.py 3 2>&1 | head -2; done
REBK_PROF=1 python tools/shard_virtual_timing.py 1 2>&1 | head -16

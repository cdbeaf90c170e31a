# stream-kernel ring depth A/B on C3 (same shared-memory budget split into NS stages)
for ns in 2 3 4 6 2; do echo "== REBK_STREAM_NS=$ns"; REBK_STREAM_NS=$ns python tools/shard_virtual_timing.py 3 2>&1 | grep -E "single"; done

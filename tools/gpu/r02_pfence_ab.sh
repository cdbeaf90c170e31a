for v in "1 2" "0 2" "0 3" "1 2" "0 2"; do set -- $v; echo "== PFENCE=$1 NS=$2"; REBK_STREAM_PFENCE=$1 REBK_STREAM_NS=$2 python tools/shard_virtual_timing.py 3 2>&1 | grep single; done
REBK_STREAM_PFENCE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "stream" 2>&1 | tail -2

for cfg in "PGCP_WELD_SPIN_NS=0" "PGCP_WELD_SPIN_NS=64" "PGCP_WELD_SPIN_NS=200" "PGCP_WELD_STREAM=0" "PGCP_WELD_STREAM=0 PGCP_WELD_SPIN_NS=100"; do
  echo "== $cfg"; env $cfg python tools/weld_timing.py 2>&1 | grep -E "weld ms|k 1023|step 56 " | tail -3
done

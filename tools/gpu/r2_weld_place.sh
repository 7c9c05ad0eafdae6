# does keeping the streamed replay's CTAs off the SMs of phase 1 help the chain?
for cfg in "PGCP_WELD_REPLAY_NT=128" "PGCP_WELD_REPLAY_NT=256" "PGCP_WELD_REPLAY_NT=512" "PGCP_WELD_REPLAY_NT=512 PGCP_WELD_REPLAY_SMEM_KB=120" "PGCP_WELD_REPLAY_NT=512 PGCP_WELD_REPLAY_SMEM_KB=200" "PGCP_WELD_REPLAY_NT=256 PGCP_WELD_REPLAY_SMEM_KB=100" "PGCP_WELD_REPLAY_NT=1024 PGCP_WELD_REPLAY_SMEM_KB=200"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/weld_stage_split.py 2>&1 | grep -E "device ms|weld stage" | tail -2
done
